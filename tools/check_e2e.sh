(timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host" 2>&1 | tail -3) > gpurun_out/pytest_host.log 2>&1
tail -2 gpurun_out/pytest_host.log
timeout 900 python bench.py --no-extras > gpurun_out/bench_e2e.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/bench_e2e.log').read().strip().splitlines()[-1])
print(d['value'], d.get('e2e'), d['roofline']['frac'], d['roofline'].get('traffic'))"
