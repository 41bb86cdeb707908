timeout 600 python tools/ab_option.py ntt_q 7 > gpurun_out/ab_quick.log 2>&1
