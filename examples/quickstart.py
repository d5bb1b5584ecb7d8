"""Encrypted embedding lookup in a few calls (one B200).

The client one-hot encodes its token and encrypts it; the server packs the
plaintext table once (hybrid diagonals, baby-step/giant-step plan) and runs
the lookup on the ciphertext; the client decrypts the embedding row.

    python examples/quickstart.py            # Tiny ring (N = 2^12)
    python examples/quickstart.py criteo     # the Criteo-shaped model (N = 2^16)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2506_18150_b200 import helrm  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tiny_a"
w = synth.make_workload(name)            # seeded synthetic tables + one query
cfg = w.config

# --- setup (server and client share the parameters) ---
params = helrm.params_from_config(cfg)   # ring, RNS primes, scale
stream = torch.cuda.Stream()
ctx = helrm.Context(params, 0, stream.cuda_stream)
tables = helrm.tables_create(params, w.tables, w.n_dense)
t0 = time.time()
plan = helrm.plan_create(ctx, tables, cfg.level)   # server: pack, pre-rotate, encode the diagonals
info = plan.info()
print(f"{name}: {info.n_diag} diagonals, {info.n_in_cts} input ct(s), {info.n_rotations} rotation keys, "
      f"plan {time.time() - t0:.1f} s")

# --- client: keys, one-hot query, encryption ---
sk = helrm.sk_gen(ctx, cfg.seed)
pk = helrm.pk_gen(ctx, sk, cfg.seed)
rk = helrm.rotkeys_gen(ctx, sk, plan.galois(cfg.N), cfg.seed)   # sent to the server once
x = helrm.encode_query(tables, w.indices[0], w.dense[0], info.n_in_cts * cfg.n_slots)
cts = [helrm.encrypt(ctx, pk, x[c * cfg.n_slots:(c + 1) * cfg.n_slots], cfg.level, (cfg.seed << 20) | c)
       for c in range(info.n_in_cts)]

# --- server: the encrypted lookup ---
for _ in range(2):   # the first call runs eagerly, the second captures the CUDA graph replayed after
    for o in helrm.lookup(ctx, plan, rk, cts):
        o.close()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
outs = helrm.lookup(ctx, plan, rk, cts)
e1.record(stream)
torch.cuda.synchronize()

# --- client: decrypt ---
y = np.concatenate([helrm.decrypt_decode(ctx, sk, o) for o in outs])
print(f"lookup {e0.elapsed_time(e1):.2f} ms; first outputs {np.round(y[:4], 5)}")
if name == "tiny_a":   # one uncompressed table: the answer is simply its row
    row = w.tables[0].weights[w.indices[0][0]]
    print(f"max |decrypted - table row| = {np.abs(y[: len(row)] - row).max():.2e}")
