# r02: tcgen05 (kind::i8) BSGS MAC: first parity check on small shapes, then the bench-shape tests + quick bench
(timeout 300 python -m pytest tests/test_gpu_edges.py -q -x -k "worst_case or degenerate" 2>&1 | tail -15) > gpurun_out/pytest_mac_tc_a.log 2>&1
(timeout 600 python -m pytest tests/test_gpu_launch_shape.py tests/test_gpu_parity.py -q -x -k "forward or bench_shape or guard" 2>&1 | tail -15) > gpurun_out/pytest_mac_tc_b.log 2>&1
timeout 600 python bench.py --no-extras --no-cpu-baseline --no-e2e --no-ks-variant > gpurun_out/bench_quick.log 2>&1
