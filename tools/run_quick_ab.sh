# one B = 256 forward chunk with per-kernel times (library probe) + the hybrid / launch-shape parity tests
set -x
timeout 600 python tools/ab_option.py ntt_q 7 > gpurun_out/ab_quick.log 2>&1
timeout 900 python -m pytest tests/test_gpu_hybrid_ks.py tests/test_gpu_launch_shape.py -m gpu -x -q > gpurun_out/pytest_quick.log 2>&1
