timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -m gpu -q -x -k "lookup or golden or batched or rotate or host or extraction or dense" > gpurun_out/r2_rs.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_rs.txt
for v in "HELRM_ROTSUM_SPLIT=0" "X=1" "HELRM_ROTSUM_SPLIT=0" "X=1"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --skip-cpu-baseline --skip-micro --skip-batch --skip-llm --skip-c2 > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json"))
print(f"{sys.argv[1]:40s} step {d['ms_per_step']:.3f} ms e2e {d['e2e']['value']}", flush=True)
PY
done
