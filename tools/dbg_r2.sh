for ch in 512 1024 2304 512 1024; do
  HELRM_NTT_CHUNK=$ch timeout 300 python bench.py --steps 20 --warmup 5 --skip-cpu-baseline --skip-micro --skip-batch --skip-llm --skip-c2 > gpurun_out/ab_tmp.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_tmp.json')); k=d['step']['kernels']; print('chunk $ch step', d['ms_per_step'], 'e2e', d['e2e']['value'], 'p1', k['ntt_fwd_p1']['ms_per_step'], 'p2', k['ntt_fwd_p2']['ms_per_step'])"
done
