# round-1 re-entry check: parity tests, smoke, full bench (+e2e, cpu baseline, sub-benchmarks),
# reference arm, and the launch list of one profiled forward chunk (B=256)
(timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30) > gpurun_out/pytest_gpu.log 2>&1
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5) > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
P="python tools/profile_forward.py"
$P --mode forward --batch 256 > gpurun_out/pf_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_forward_b256.csv $P --mode forward --batch 256 > gpurun_out/ncu1.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -n 1 gpurun_out/bench_full.log gpurun_out/bench_ref.log
