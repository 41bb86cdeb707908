# r02: new parity/edge tests, then the full bench (extras, latency, cpu_baseline + parity leg)
set -x
(timeout 1500 python -m pytest tests/test_gpu_launch_shape.py tests/test_gpu_edges.py -q 2>&1 | tail -25) > gpurun_out/pytest_new.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_full.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_full.log
