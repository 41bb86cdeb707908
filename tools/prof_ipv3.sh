# ncu --set full of one k_ks_ip_mma3 launch (B = 256 dense1 chunk)
P="python tools/profile_forward.py --mode forward --batch 256"
$P > gpurun_out/pf.log 2>&1 &&
ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_ks_ip_mma3" -c 1 -o gpurun_out/prof_ipv3 $P > gpurun_out/ncu_ipv3.log 2>&1
ncu -i gpurun_out/prof_ipv3.ncu-rep --page raw --csv > gpurun_out/prof_ipv3_raw.csv 2>&1
ncu -i gpurun_out/prof_ipv3.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_ipv3_source.csv 2>&1
gzip -f gpurun_out/prof_ipv3_source.csv
rm -f gpurun_out/prof_ipv3.ncu-rep
