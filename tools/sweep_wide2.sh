# NTT thread-count sweep (CKKS_NTT_WIDE bit mask: 1 digits, 2 ModUp, 4 ModDown iNTT, 8 ModDown NTT)
for m in 2 0 3 6 10; do
  CKKS_NTT_WIDE=$m timeout 600 python bench.py --no-cpu-baseline --no-extras --no-e2e > gpurun_out/bench_w$m.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_w$m.log').read().strip().splitlines()[-1]);print($m,d['value'],{k:v['ms_per_step'] for k,v in d['kernel_shares'].items() if k in ('k_ks_modup','k_ks_digits','k_ks_moddown_ntt','k_ks_moddown_intt','k_ks_qp_rem')})"
done
