# parity subset + A/B of the key-stationary giant-step IP (CKKS_IP_GIANT=1 default vs 0)
(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_frozen_stack.py tests/test_gpu_edges.py -x -q -k "hoist or stack or forward or edge or level or worst or host" 2>&1 | tail -3) > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
for m in 1 0; do
  CKKS_IP_GIANT=$m timeout 600 python bench.py --no-cpu-baseline --no-extras --no-e2e > gpurun_out/bench_giant$m.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_giant$m.log').read().strip().splitlines()[-1]);print($m,d['value'],{k:v['ms_per_step'] for k,v in list(d['kernel_shares'].items())[:8]})"
done
