timeout 1500 python -m pytest tests -m gpu -q -x -k "not (llm_full or c2_full)" > gpurun_out/r2_t2_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_t2_pytest.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_t2_bench.json 2> gpurun_out/r2_t2_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/r2_t2_bench.err
