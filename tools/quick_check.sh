# parity subset + one bench line (default options); usage: bash tools/quick_check.sh [pytest -k expr]
K=${1:-"hoist or stack or conv or degenerate"}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_frozen_stack.py tests/test_gpu_edges.py -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-extras > gpurun_out/bench.log 2>&1
tail -c 3000 gpurun_out/bench.log
