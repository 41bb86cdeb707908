# parity subset covering the BSGS MAC + one bench line
(timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15) > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-extras --no-e2e > gpurun_out/bench.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]);print(d['value'],{k:v['ms_per_step'] for k,v in list(d['kernel_shares'].items())[:8]})"
