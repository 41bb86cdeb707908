# worst-case MAC/IP exactness test + ncu capture (dram traffic) of the merged baby-step IP kernel
(timeout 900 python -m pytest tests/test_gpu_edges.py -x -q 2>&1 | tail -5) > gpurun_out/pytest_edges.log 2>&1
tail -2 gpurun_out/pytest_edges.log
P="python tools/profile_forward.py --mode forward --batch 256"
$P > gpurun_out/pf.log 2>&1 || exit 1
for spec in "k_ks_ip_mma2<.int.8>:ipmma2" "k_bsgs_mac_mma<.bool.0:macmma_fp"; do
  re=${spec%%:*}; tag=${spec##*:}
  ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$re" -c 1 -o gpurun_out/prof_$tag $P > gpurun_out/ncu_$tag.log 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_source.csv 2>&1
  gzip -f gpurun_out/prof_${tag}_source.csv
  rm -f gpurun_out/prof_$tag.ncu-rep
done
ls -la gpurun_out | grep prof_
