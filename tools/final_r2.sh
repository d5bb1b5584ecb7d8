#!/bin/bash
# End-of-round ncu captures: the launch list of one lookup step and one ncu --set full capture
# of the same step (per-kernel DRAM traffic for bench.py's roofline.traffic).  The bench line
# itself: python bench.py --steps 20 --warmup 5 --with-compact (separate call).
set -u
timeout 600 python bench.py --ncu-step --warmup 3 --skip-cpu-baseline > gpurun_out/r2_final_ncustep_plain.log 2>&1; rc=$?; echo "ncu-step plain rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu -f --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/r2_final_launches.csv python bench.py --ncu-step --warmup 3 --skip-cpu-baseline > gpurun_out/r2_final_ncu_launch.log 2>&1
  echo "launch list rc=$?"
  timeout 1800 ncu -f --set full --clock-control none --import-source on --profile-from-start off -o /tmp/r2_full \
    python bench.py --ncu-step --warmup 3 --skip-cpu-baseline > gpurun_out/r2_final_ncu_full.log 2>&1
  echo "ncu full rc=$?"
  python tools/ncu_traffic.py /tmp/r2_full.ncu-rep > gpurun_out/r2_final_ncu_traffic.json 2>&1
  python tools/ncu_summary.py /tmp/r2_full.ncu-rep 400 > gpurun_out/r2_final_ncu_full_summary.txt 2>&1
  python tools/launch_summary.py gpurun_out/r2_final_launches.csv > gpurun_out/r2_final_launch_summary.txt 2>&1
fi
