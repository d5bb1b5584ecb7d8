timeout 2400 python -m pytest tests -m gpu -q -x -k "not llm_full" > gpurun_out/r2_t5_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_t5_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
