# r02 first GPU call: the new launch-shape parity tests, the full GPU suite, compute-sanitizer on the
# cp.async / smem kernels at B = 33, a short bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
(timeout 1500 python -m pytest tests/test_gpu_launch_shape.py -q -x 2>&1 | tail -15) > gpurun_out/pytest_launch_shape.log 2>&1
(timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15) > gpurun_out/pytest_gpu.log 2>&1
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_forward.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_$tool.log
done
timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1
