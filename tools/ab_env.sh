#!/bin/bash
# A/B timing of env-switched variants: ./tools/ab_env.sh "ENV1=.. ENV2=.." "..."
for v in "$@"; do
  env $v python bench.py --steps 10 --warmup 3 --skip-cpu-baseline --skip-micro --skip-batch --skip-llm --skip-c2 > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json"))
print(f"{sys.argv[1]:50s} step {d['ms_per_step']:.3f} ms  ({d['value']} lookups/s, e2e {d['e2e']['value']})")
PY
done
