# A/B of the giant-step inner product batch per thread (CKKS_IPQ_BB = 2 default, 4, 1)
for m in 2 4 1; do
  CKKS_IPQ_BB=$m timeout 600 python bench.py --no-cpu-baseline --no-extras --no-e2e > gpurun_out/bench_bb$m.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_bb$m.log').read().strip().splitlines()[-1]);print($m,d['value'],{k:v['ms_per_step'] for k,v in list(d['kernel_shares'].items())[:4]})"
done
