# chunk size A/B: ciphertexts per internal launch sequence
for mb in 512 256; do
  timeout 600 python bench.py --no-cpu-baseline --no-extras --no-e2e --max-batch $mb > gpurun_out/bench_mb$mb.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_mb$mb.log').read().strip().splitlines()[-1]);print($mb,d['value'],{k:v['ms_per_step'] for k,v in list(d['kernel_shares'].items())[:8]})" || tail -5 gpurun_out/bench_mb$mb.log
done
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
