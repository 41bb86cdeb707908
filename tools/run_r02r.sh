set -x
timeout 600 python tools/ntt_q_check.py > gpurun_out/ntt_c_check2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_fpr.log 2>&1
