timeout 900 python -m pytest tests/test_gpu_boundary.py -m gpu -q -x -k "hoisted_batch" > gpurun_out/r2_rotb.txt 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2_rotb.txt
timeout 600 python bench.py --steps 3 --warmup 3 --skip-cpu-baseline --skip-batch --skip-llm --skip-c2 > gpurun_out/r2_micro.json 2>/dev/null; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r2_micro.json')); s=d['secondary']; print({k: s[k] for k in s if 'rot' in k or 'ntt' in k})"
