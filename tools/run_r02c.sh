# r02: hybrid key switching (f-3) parity + the full GPU suite (regression of the K = 1 path)
(timeout 1500 python -m pytest tests/test_gpu_hybrid_ks.py -q -x 2>&1 | tail -30) > gpurun_out/pytest_hybrid.log 2>&1
(timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_hybrid_ks.py 2>&1 | tail -30) > gpurun_out/pytest_gpu_all.log 2>&1
