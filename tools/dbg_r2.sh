timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline --skip-micro --skip-llm --skip-c2 --skip-batch > gpurun_out/r2_t3_bench.json 2> gpurun_out/r2_t3_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2_t3_bench.json"))
print(d["value"], d["ms_per_step"], d["e2e"]["value"])
for k, v in d["step"]["kernels"].items(): print(f"{k:14s} {v}")
PY
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 1 python tools/sanitize_case.py > gpurun_out/r2_memcheck.txt 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/r2_memcheck.txt
