timeout 900 python bench.py --max-batch 512 --no-extras --no-cpu-baseline --no-e2e --no-ks-variant > gpurun_out/bench_mb512.log 2>&1
timeout 900 python bench.py --max-batch 256 --no-extras --no-cpu-baseline --no-e2e --no-ks-variant > gpurun_out/bench_mb256.log 2>&1
