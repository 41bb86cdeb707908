(timeout 900 python -m pytest tests/test_gpu_launch_shape.py tests/test_gpu_edges.py -q -x -k "mac_tensor or worst_case" 2>&1 | tail -5) > gpurun_out/pytest_mactc.log 2>&1
(timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -15) > gpurun_out/pytest_gpu_all.log 2>&1
