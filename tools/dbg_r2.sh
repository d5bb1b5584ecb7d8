timeout 600 python bench.py --steps 3 --warmup 3 --skip-cpu-baseline --skip-micro --skip-c2 > gpurun_out/r2_b64.json 2>/dev/null; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r2_b64.json')); s=d['secondary']
for k in ('criteo_b64','llm_128_tokens'): print(k, json.dumps({kk: s[k][kk] for kk in s[k] if kk in ('ms_per_batch','ms_per_lookup','fp64_frac_model','profiled_kernel_ms','ntt_limb_transforms_per_run')}))"
