# r02: quick bench (hybrid headline + single variant) after specialising the KS NTT kernels; hybrid parity
(timeout 900 python -m pytest tests/test_gpu_hybrid_ks.py -q -x 2>&1 | tail -5) > gpurun_out/pytest_hybrid.log 2>&1
timeout 900 python bench.py --no-extras --no-cpu-baseline --no-e2e > gpurun_out/bench_quick.log 2>&1
