P="python tools/profile_forward.py --mode forward --batch 256"
ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base function -k k_ks_ip_giant_multi -c 1 -o gpurun_out/prof_ipgm $P > gpurun_out/ncu_ipgm.log 2>&1
ncu -i gpurun_out/prof_ipgm.ncu-rep --page raw --csv > gpurun_out/prof_ipgm_raw.csv 2>&1
ncu -i gpurun_out/prof_ipgm.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_ipgm_source.csv 2>&1
gzip -f gpurun_out/prof_ipgm_source.csv
rm -f gpurun_out/prof_ipgm.ncu-rep
