# bench with different CKKS_NTT_WIDE masks (tuning experiment)
for m in "$@"; do
  CKKS_NTT_WIDE=$m timeout 300 python bench.py --no-cpu-baseline --no-extras --no-e2e --steps 2 > gpurun_out/sweep_$m.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/sweep_$m.log').read().strip().splitlines()[-1])
print('mask $m', d['value'], {k: v['ms_per_step'] for k,v in d['kernel_shares'].items() if v['share']>0.02})"
done
