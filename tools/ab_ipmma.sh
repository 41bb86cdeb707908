timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_frozen_stack.py -x -q -k "hoist or stack" > gpurun_out/pytest_gpu.log 2>&1
for m in 1 0; do
  CKKS_IP_MMA=$m timeout 600 python bench.py --no-cpu-baseline --no-extras --no-e2e > gpurun_out/bench_mma$m.log 2>&1
done
python tools/profile_forward.py --mode forward --batch 256 > gpurun_out/pf.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_ks_ip_mma -c 1 -o gpurun_out/prof_ipmma python tools/profile_forward.py --mode forward --batch 256 > gpurun_out/ncu_ipmma.log 2>&1
ncu -i gpurun_out/prof_ipmma.ncu-rep --page raw --csv > gpurun_out/prof_ipmma_raw.csv 2>&1
ncu -i gpurun_out/prof_ipmma.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_ipmma_source.csv 2>&1
gzip -f gpurun_out/prof_ipmma_source.csv; rm -f gpurun_out/prof_ipmma.ncu-rep
