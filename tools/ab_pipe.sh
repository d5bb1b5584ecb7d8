# A/B of the giant-step pipeline with a smaller bulk-MAC ring (co-residence of NTT and MAC CTAs)
for v in "HELRM_PIPE=0" "HELRM_PIPE=1" "HELRM_PIPE=1 HELRM_MACB_STAGES=6" "HELRM_PIPE=1 HELRM_MACB_STAGES=6 HELRM_MACCH=1 HELRM_NTTCH=4" "HELRM_PIPE=1 HELRM_MACB_STAGES=8 HELRM_MACCH=2 HELRM_NTTCH=8" "HELRM_PIPE=1 HELRM_MACB_STAGES=4 HELRM_MACCH=1 HELRM_NTTCH=4" "HELRM_PIPE=0 HELRM_MACB_STAGES=6"; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline --skip-micro --skip-batch --skip-llm --skip-c2 > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json"))
print(f"{sys.argv[1]:75s} step {d['ms_per_step']:.3f} ms  ({d['value']} lookups/s, e2e {d['e2e']['value']})", flush=True)
PY
done
