# per-kernel times of the cluster ModUp at N = 16384 (option ntt_q bit 8) inside one B = 256 forward chunk
CKKS_NTT_Q=15 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ks_modup -c 60 --csv --log-file gpurun_out/launches_modupc.csv python tools/ab_option.py ntt_q 15 --reps 1 > gpurun_out/ncu_modupc.log 2>&1
