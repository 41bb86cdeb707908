# parity subset + bench: 60-bit IP rows on IMAD (overlapping the DMMA rows), NTT batch forward wide
(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_frozen_stack.py tests/test_gpu_edges.py -x -q -k "hoist or stack or forward or edge or level or worst or host or ntt" 2>&1 | tail -3) > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_ii.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_ii.log').read().strip().splitlines()[-1]);print(d['value'],{k:v['ms_per_step'] for k,v in list(d['kernel_shares'].items())[:8]}, d['ntt_microbench']['fwd'], d['frozen_stack_p2']['forwards_per_s'])"
