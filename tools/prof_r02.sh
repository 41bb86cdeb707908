# r02 profiling of the hybrid forward (B=256 chunk): launch list + ncu --set full of the top kernels
P="python tools/profile_forward.py --mode forward --batch 256"
$P > gpurun_out/pf.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_forward_b256.csv $P > gpurun_out/ncu1.log 2>&1
for spec in "k_ks_modup<14, 512, 2>:modup2" "k_ks_modup<14, 512, 1>:modup1" "k_ks_ip_mma2:ipmma2" "k_bsgs_mac_mma:macmma" "k_ks_digits<14, 1024, 2, 0>:digits2"; do
  re=${spec%%:*}; tag=${spec##*:}
  ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$re" -c 1 -o gpurun_out/prof_$tag $P > gpurun_out/ncu_$tag.log 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_source.csv 2>&1
  gzip -f gpurun_out/prof_${tag}_source.csv
  rm -f gpurun_out/prof_$tag.ncu-rep
done
