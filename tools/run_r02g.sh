# r02: full GPU suite (new client / p1 / graph tests) + full bench
(timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -30) > gpurun_out/pytest_gpu_all.log 2>&1
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5) > gpurun_out/smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_full.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_full.log
