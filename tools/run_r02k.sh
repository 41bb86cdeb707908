# r02 re-entry: full GPU suite + smoke + default bench on the restored tree
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
(timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -15) > gpurun_out/pytest_gpu_all.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
