timeout 600 python tools/ab_option.py ip_v3 0 1 > gpurun_out/ab_ipv3.log 2>&1
(timeout 1800 python -m pytest tests/test_gpu_launch_shape.py tests/test_gpu_hybrid_ks.py tests/test_gpu_edges.py -x -q 2>&1 | tail -15) > gpurun_out/pytest_ipv3.log 2>&1
