#!/bin/bash
for v in "$@"; do
  env $v python bench.py --steps 5 --warmup 3 --skip-cpu-baseline --skip-batch --skip-llm --skip-c2 --rot-cts 2 > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json"))
k = d["step"]["kernels"]
f = lambda n: k.get(n, {}).get("ms_per_step", 0)
print(f"{sys.argv[1][-40:]:40s} step {d['ms_per_step']:.3f} ms | p1 {f('ntt_fwd_p1'):.3f} p2 {f('ntt_fwd_p2'):.3f} pa {f('ntt_inv_pa'):.3f} pb {f('ntt_inv_pb'):.3f} conv {f('conv'):.3f} | micro fwd {d['secondary']['ntt_fwd_GBps']} inv {d['secondary']['ntt_inv_GBps']} GB/s")
PY
done
