"""The 17-input-ct Criteo shape (Table 2's 10^2x model analog:
535,963 one-hot slots, 8704 diagonals, ~119 GiB of QP-NTT plaintexts in HBM)
on one B200: plan counts, decryption against the float64 gather and the
batch-1 lookup time.  Too large for the test suite's shared process; run
alone:  python tests/manual/c17_check.py > profiles/<round>_c17.txt"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from oracle import lookup as lk  # noqa: E402  (test infrastructure: the float64 gather only)
from paper_2506_18150_b200 import helrm  # noqa: E402

w = synth.make_workload("criteo_c17")
cfg = w.config
P = helrm.params_from_config(cfg)
stream = torch.cuda.Stream()
ctx = helrm.Context(P, 0, stream.cuda_stream)
t0 = time.time()
T = helrm.tables_create(P, w.tables, w.n_dense)
plan = helrm.plan_create(ctx, T, cfg.level)
info = plan.info()
sk = helrm.sk_gen(ctx, cfg.seed)
pk = helrm.pk_gen(ctx, sk, cfg.seed)
rk = helrm.rotkeys_gen(ctx, sk, plan.galois(cfg.N), cfg.seed)
x = helrm.encode_query(T, w.indices[0], w.dense[0], info.n_in_cts * cfg.n_slots)
cts = [helrm.encrypt(ctx, pk, x[c * cfg.n_slots:(c + 1) * cfg.n_slots], cfg.level, (cfg.seed << 20) | c)
       for c in range(info.n_in_cts)]
ctx.sync()
print(f"setup {time.time() - t0:.1f} s: {info.n_in_cts} input cts, {info.n_diag} diagonals, "
      f"{info.diag_bytes / 2**30:.1f} GiB plaintexts, {rk.nbytes() / 2**30:.2f} GiB keys, n1={info.n1}, "
      f"rotations={info.n_rotations}", flush=True)
outs = helrm.lookup(ctx, plan, rk, cts)
z = helrm.decrypt_decode(ctx, sk, outs[0])
lay = lk.layout(w)
err = float(np.abs(z[: lay.M] - lk.gather(lay, w.indices[0])).max())
for o in outs:
    o.close()
print(f"decrypted vs float64 gather: max abs err {err:.2e} ({'ok' if err < 1e-3 else 'FAIL'})", flush=True)
for _ in range(2):
    for o in helrm.lookup(ctx, plan, rk, cts):
        o.close()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record(stream)
for _ in range(reps):
    for o in helrm.lookup(ctx, plan, rk, cts):
        o.close()
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"batch-1 lookup: {ms:.2f} ms ({1e3 / ms:.1f} lookups/s); the paper's CPU embedding for its 18-ct model: "
      f"44-51 s (PAPER.md:472-475)", flush=True)
free, total = torch.cuda.mem_get_info()
print(f"device memory in use at the end: {(total - free) / 2**30:.1f} GiB of {total / 2**30:.1f} GiB")
sys.exit(0 if err < 1e-3 else 1)
