# full GPU parity + bench with the sub-benchmarks (cfg2 NTT on 50-bit primes, p2 frozen stack)
(timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15) > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_fpr.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/bench_fpr.log').read().strip().splitlines()[-1])
print(d['value'], d.get('e2e',{}).get('value'), d['ntt_microbench']['fwd'], d['ntt_microbench']['inv'], d['frozen_stack_p2']['forwards_per_s'], d['keyswitch']['rotations_per_s'])"
