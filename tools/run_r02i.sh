(timeout 300 python -m pytest tests/test_gpu_edges.py -q -x -k "worst_case or degenerate" 2>&1 | tail -3) > gpurun_out/pytest_mac_tc_a.log 2>&1
timeout 600 python bench.py --no-extras --no-cpu-baseline --no-e2e --no-ks-variant > gpurun_out/bench_quick.log 2>&1
bash tools/prof_one_kernel.sh k_bsgs_mac_tc mactc 0
bash tools/prof_one_kernel.sh k_ks_ip_mma2 ipmma2 0
