# r02 session 3: evidence on the restored tree (ip_v3 default): GPU suite, smoke, bench, launch list,
# ncu --set full of the NTT kernels (ModUp, digits), the ip_v3 IP and the cfg2 batch NTT
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
(timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -15) > gpurun_out/pytest_gpu_all.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
P="python tools/profile_forward.py --mode forward --batch 256"
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_forward_b256.csv $P > gpurun_out/ncu1.log 2>&1
for spec in "k_ks_modup<14, 512, 2>:modup2" "k_ks_ip_mma3:ipmma3" "k_ks_digits<14, 1024, 2, 0>:digits2"; do
  re=${spec%%:*}; tag=${spec##*:}
  ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$re" -c 1 -o gpurun_out/prof_$tag $P > gpurun_out/ncu_$tag.log 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_source.csv 2>&1
  gzip -f gpurun_out/prof_${tag}_source.csv
  rm -f gpurun_out/prof_$tag.ncu-rep
done
P2="python tools/profile_forward.py --mode ntt"
ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_ntt_batch" -c 2 -o gpurun_out/prof_nttbatch $P2 > gpurun_out/ncu_nttbatch.log 2>&1
ncu -i gpurun_out/prof_nttbatch.ncu-rep --page raw --csv > gpurun_out/prof_nttbatch_raw.csv 2>&1
ncu -i gpurun_out/prof_nttbatch.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_nttbatch_source.csv 2>&1
gzip -f gpurun_out/prof_nttbatch_source.csv
rm -f gpurun_out/prof_nttbatch.ncu-rep
