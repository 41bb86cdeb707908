(timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg3 or hoisted_parity" 2>&1 | tail -3) > gpurun_out/pytest_cfg3.log 2>&1
tail -2 gpurun_out/pytest_cfg3.log
python - <<PY
import sys, argparse; sys.path.insert(0, '.')
import torch, bench, synthetic as S
from paper_2205_11935_b200 import ckks as G
print(bench.bench_keyswitch(G, S, torch.device('cuda', 0), argparse.Namespace(steps=3)))
PY
