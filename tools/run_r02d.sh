# r02: bench with the hybrid key switching headline (+ the single variant as a sub-line)
timeout 1500 python bench.py > gpurun_out/bench_hybrid.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_hybrid.log
