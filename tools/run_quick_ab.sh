timeout 600 python tools/ab_option.py ntt_q 15 > gpurun_out/ab_quick.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_launch_shape.py tests/test_gpu_hybrid_ks.py tests/test_gpu_edges.py -m gpu -x -q > gpurun_out/pytest_quick.log 2>&1
