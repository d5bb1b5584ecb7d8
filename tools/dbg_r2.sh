timeout 1200 python -m pytest tests/test_gpu_boundary.py -m gpu -q -x -k "limb" > gpurun_out/r2_limb.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2_limb.txt
