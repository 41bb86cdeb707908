timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hoist" > gpurun_out/pytest_gpu.log 2>&1
CKKS_IP_MMA=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_frozen_stack.py -x -q -k "hoist or stack" > gpurun_out/pytest_gpu_mma.log 2>&1
for m in 1 0; do
  CKKS_IP_MMA=$m timeout 600 python bench.py --no-cpu-baseline --no-extras --no-e2e > gpurun_out/bench_mma$m.log 2>&1
done
