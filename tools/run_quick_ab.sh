set -x
timeout 900 python tools/ab_p1.py ntt_q 0 15 > gpurun_out/ab_p1.log 2>&1
timeout 600 python tools/ntt_q_check.py > gpurun_out/ntt_c_check3.log 2>&1
