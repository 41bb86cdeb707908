set -x
timeout 600 python tools/ntt_q_check.py > gpurun_out/ntt_c_check.log 2>&1
timeout 900 python tools/ab_p1.py ntt_q 0 3 7 > gpurun_out/ab_nttc_p1.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_nttc.log 2>&1
