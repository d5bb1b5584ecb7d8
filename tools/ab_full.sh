#!/bin/bash
# A/B of env variants on b1 + batch 64 + LLM (no CPU baseline, no microbenchmarks)
for v in "$@"; do
  env $v python bench.py --steps 5 --warmup 3 --skip-cpu-baseline --skip-micro > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json"))
s = d["secondary"]
k = d["step"]["kernels"]
f = lambda n: k.get(n, {}).get("ms_per_step", 0)
print(f"{sys.argv[1][-40:]:40s} b1 {d['ms_per_step']:.3f} ms ({d['value']}/s, e2e {d['e2e']['value']}) mac {f('diag_mac'):.3f} | b64 {s['criteo_b64']['lookups_per_s']}/s | llm {s['llm_128_tokens']['token_lookups_per_s']} tok/s")
PY
done
