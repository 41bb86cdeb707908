# round-end evidence: parity, smoke, full bench (+e2e, cpu baseline, sub-benchmarks), reference arm,
# launch list of one profiled forward chunk (B=256), ncu --set full of the top kernels
(timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15) > gpurun_out/pytest_gpu.log 2>&1
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5) > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
P="python tools/profile_forward.py --mode forward --batch 256"
$P > gpurun_out/pf.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_forward_b256.csv $P > gpurun_out/ncu1.log 2>&1
for spec in "k_ks_ip_mma2<.int.8>:ipmma2" "k_bsgs_mac_mma:macmma" "k_ks_modup<.int.14:modup" "k_ks_ip_giant<.int.8>:ipgiant"; do
  re=${spec%%:*}; tag=${spec##*:}
  ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$re" -c 1 -o gpurun_out/prof_$tag $P > gpurun_out/ncu_$tag.log 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_source.csv 2>&1
  gzip -f gpurun_out/prof_${tag}_source.csv
  rm -f gpurun_out/prof_$tag.ncu-rep
done
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 600 gpurun_out/bench_full.log; tail -c 300 gpurun_out/bench_ref.log
