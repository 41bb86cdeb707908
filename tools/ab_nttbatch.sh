# cfg2 batched NTT: 16 (default) vs 32 residues per thread (CKKS_NTT_WIDE bit 16)
for m in 2 18; do
  CKKS_NTT_WIDE=$m python - <<PY
import sys, argparse; sys.path.insert(0, '.')
import torch, bench, synthetic as S
from paper_2205_11935_b200 import ckks as G
a = argparse.Namespace(steps=10)
print($m, bench.bench_ntt(G, S, torch.device('cuda', 0), a))
PY
done
(timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ntt" 2>&1 | tail -2)
CKKS_NTT_WIDE=18 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ntt" 2>&1 | tail -2
