# A/B of the BSGS MAC on the FP64 tensor cores (CKKS_MAC_MMA=1, default) vs the DFMA/int128 kernels
(timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15) > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for m in 1 0; do
  CKKS_MAC_MMA=$m timeout 600 python bench.py --no-cpu-baseline --no-extras --no-e2e > gpurun_out/bench_macmma$m.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_macmma$m.log').read().strip().splitlines()[-1]);print($m,d['value'],{k:v['ms_per_step'] for k,v in list(d['kernel_shares'].items())[:7]})"
done
[ -x tools/pipe_bench ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_bench tools/pipe_bench.cu
(timeout 120 ./tools/pipe_bench 2>&1 | tail -20) > gpurun_out/pipe_bench.log 2>&1; cat gpurun_out/pipe_bench.log
