set -x
timeout 600 python tools/ntt_q_check.py > gpurun_out/ntt_q_check.log 2>&1
timeout 600 python tools/ab_option.py ntt_q 0 4 > gpurun_out/ab_nttq_modup.log 2>&1
