# round-end evidence (short form): parity, smoke, full bench, reference arm, launch list, ncu --set full of the top two kernels
(timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15) > gpurun_out/pytest_gpu.log 2>&1
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5) > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
P="python tools/profile_forward.py --mode forward --batch 256"
$P > gpurun_out/pf.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_forward_b256.csv $P > gpurun_out/ncu1.log 2>&1
for spec in "k_ks_ip_mma2<.int.8>:ipmma2" "k_ks_modup<.int.14:modup"; do
  re=${spec%%:*}; tag=${spec##*:}
  ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$re" -c 1 -o gpurun_out/prof_$tag $P > gpurun_out/ncu_$tag.log 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_source.csv 2>&1
  gzip -f gpurun_out/prof_${tag}_source.csv
  rm -f gpurun_out/prof_$tag.ncu-rep
done
