python bench.py --steps 2 --warmup 3 --ncu-step --skip-cpu-baseline > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --ncu-step --skip-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo "launch list rc=$?"
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_ntt|k_diag_mac|k_kip|k_conv" -o /tmp/r02_full python bench.py --steps 2 --warmup 3 --ncu-step --skip-cpu-baseline > gpurun_out/ncu_f.log 2>&1; echo "full rc=$?"
python tools/ncu_traffic.py /tmp/r02_full.ncu-rep > gpurun_out/r02_ncu_traffic.json
python tools/ncu_summary.py /tmp/r02_full.ncu-rep 200 > gpurun_out/r02_ncu_full_summary.txt
ls -la gpurun_out/
