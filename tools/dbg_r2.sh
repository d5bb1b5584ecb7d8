set -x
for p in 0 1; do HELRM_NTT_PIPE=$p timeout 120 python tools/prof_ntt.py 3072 5; done
HELRM_NTT_PIPE=0 timeout 120 python tools/prof_ntt.py 1536 1 && \
HELRM_NTT_PIPE=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ntt_fwd -s 4 -c 2 -o gpurun_out/r2_ntt_old python tools/prof_ntt.py 1536 1 > gpurun_out/r2_ncu_ntt.log 2>&1
echo "rc=$?"
