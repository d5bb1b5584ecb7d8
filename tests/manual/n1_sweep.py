"""BSGS split sweep (n1 = 32 / 64 / 16) of the Criteo batch-1 lookup on one B200: time and the
decrypted output against the float64 gather (test infrastructure: the gather is the oracle's).
Run alone:  python tests/manual/n1_sweep.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, numpy as np
import synth
from paper_2506_18150_b200 import helrm
w = synth.make_workload("criteo")
cfg = w.config
P = helrm.params_from_config(cfg)
stream = torch.cuda.Stream()
ctx = helrm.Context(P, 0, stream.cuda_stream)
T = helrm.tables_create(P, w.tables, w.n_dense)
sk = helrm.sk_gen(ctx, cfg.seed)
pk = helrm.pk_gen(ctx, sk, cfg.seed)
from oracle import lookup as lk
lay = lk.layout(w)
y = lk.gather(lay, w.indices[0])
for n1 in [32, 64, 16]:
    plan = helrm.plan_create(ctx, T, cfg.level, n1, 0)
    info = plan.info()
    rk = helrm.rotkeys_gen(ctx, sk, plan.galois(cfg.N), cfg.seed)
    x = helrm.encode_query(T, w.indices[0], w.dense[0], info.n_in_cts * cfg.n_slots)
    cts = [helrm.encrypt(ctx, pk, x, cfg.level, (cfg.seed << 20))]
    for _ in range(3):
        outs = helrm.lookup(ctx, plan, rk, cts)
        z = helrm.decrypt_decode(ctx, sk, outs[0])
        for o in outs: o.close()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        for o in helrm.lookup(ctx, plan, rk, cts): o.close()
    e1.record(stream); torch.cuda.synchronize()
    print(f"n1={n1} n2={info.n2_max} keys={info.n_rotations} ms={e0.elapsed_time(e1)/10:.3f} err={np.abs(z[:lay.M]-y).max():.2e}", flush=True)
    rk.close(); plan.close()
