timeout 1200 python -m pytest tests/test_gpu_boundary.py -m gpu -q -x -k "limb" > gpurun_out/r2_limb.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_limb.txt
timeout 900 python - <<'PY'
import sys, json
sys.argv = ["bench.py"]
import torch, synth, bench
from paper_2506_18150_b200 import helrm
w = synth.make_workload("criteo", batch=1); cfg = w.config
P = helrm.params_from_config(cfg); stream = torch.cuda.Stream(); ctx = helrm.Context(P, 0, stream.cuda_stream)
T = helrm.tables_create(P, w.tables, w.n_dense); plan = helrm.plan_create(ctx, T, cfg.level)
sk = helrm.sk_gen(ctx, cfg.seed); pk = helrm.pk_gen(ctx, sk, cfg.seed); rk = helrm.rotkeys_gen(ctx, sk, plan.galois(), cfg.seed)
x = helrm.encode_query(T, w.indices[0], w.dense[0], cfg.n_slots)
cts = [helrm.encrypt(ctx, pk, x, cfg.level, (cfg.seed << 20))]
# bit-exactness of the graph-replayed virtual form across repeated calls
ref = [helrm.ct_export(ctx, o) for o in helrm.lookup(ctx, plan, rk, cts)]
for it in range(4):
    got = [helrm.ct_export(ctx, o) for o in helrm.lookup_limbsplit_virtual(ctx, plan, rk, cts, 4)]
    print("replay", it, all((a == b).all() for a, b in zip(got, ref)))
print(json.dumps(bench.limb_split_projection(ctx, helrm, torch, stream, plan, rk, cts, cfg, (1, 2, 4, 8))["per_parts"], indent=1))
PY
