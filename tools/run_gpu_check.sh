# parity tests, bench, launch list of one profiled forward chunk (B=256)
(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30) > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
P="python tools/profile_forward.py"
$P --mode forward --batch 256 > gpurun_out/pf_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_forward_b256.csv $P --mode forward --batch 256 > gpurun_out/ncu1.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 1 gpurun_out/bench.log
