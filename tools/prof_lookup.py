"""Per-kernel breakdown (CUDA events per launch, helrm_ctx_profile) of a
Criteo lookup at a given batch:  python tools/prof_lookup.py [batch] [pipe]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2506_18150_b200 import helrm  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
name = sys.argv[2] if len(sys.argv) > 2 else "criteo"
w = synth.make_workload(name, batch=2)
cfg = w.config
P = helrm.params_from_config(cfg)
stream = torch.cuda.Stream()
ctx = helrm.Context(P, 0, stream.cuda_stream)
T = helrm.tables_create(P, w.tables, w.n_dense)
plan = helrm.plan_create(ctx, T, cfg.level)
sk = helrm.sk_gen(ctx, cfg.seed)
pk = helrm.pk_gen(ctx, sk, cfg.seed)
rk = helrm.rotkeys_gen(ctx, sk, plan.galois(cfg.N), cfg.seed)
info = plan.info()
C = info.n_in_cts
cts = []
for q in range(2):
    x = helrm.encode_query(T, w.indices[q], w.dense[q], C * cfg.n_slots)
    cts.append([helrm.encrypt(ctx, pk, x[c * cfg.n_slots:(c + 1) * cfg.n_slots], cfg.level, (cfg.seed << 20) | (q * C + c))
                for c in range(C)])
batch = [ct for i in range(B) for ct in cts[i % 2]]
for _ in range(2):
    for o in helrm.lookup(ctx, plan, rk, batch, B):
        o.close()
torch.cuda.synchronize()
import time  # noqa: E402
for rep in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    t0 = time.perf_counter()
    outs = helrm.lookup(ctx, plan, rk, batch, B)
    th = (time.perf_counter() - t0) * 1e3
    b.record(stream)
    torch.cuda.synchronize()
    for o in outs:
        o.close()
    print(f"  call {rep}: device {a.elapsed_time(b):.2f} ms, host {th:.2f} ms")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
t0 = time.perf_counter()
outs = helrm.lookup(ctx, plan, rk, batch, B)
host_ms = (time.perf_counter() - t0) * 1e3
e1.record(stream)
torch.cuda.synchronize()
for o in outs:
    o.close()
ms = e0.elapsed_time(e1)
print(f"host enqueue {host_ms:.2f} ms for one call")
ctx.profile(True)
for o in helrm.lookup(ctx, plan, rk, batch, B):
    o.close()
st = ctx.profile_stats()
ctx.profile(False)
tot = sum(v["ms"] for v in st.values())
print(f"batch {B}: {ms:.2f} ms per call, {ms / B:.3f} ms per query; profiled kernel sum {tot:.2f} ms")
for k, v in sorted(st.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"  {k:14s} {v['count']:6d} launches {v['ms']:9.3f} ms  {v['ms'] / B:8.3f} ms/query  "
          f"{v['bytes'] / max(v['ms'], 1e-9) / 1e6:8.1f} GB/s")
