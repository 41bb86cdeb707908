# usage: bash tools/prof_one.sh <kernel-regex> <tag>   (one ncu --set full capture of the first launch in a profiled forward)
P="python tools/profile_forward.py"
$P --mode forward --batch 256 > gpurun_out/pf_plain.log 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$1 -c 1 -o gpurun_out/prof_$2 $P --mode forward --batch 256 > gpurun_out/ncu_$2.log 2>&1
ncu -i gpurun_out/prof_$2.ncu-rep --page raw --csv > gpurun_out/prof_$2_raw.csv 2>&1
ncu -i gpurun_out/prof_$2.ncu-rep --page details --csv > gpurun_out/prof_$2_details.csv 2>&1
ncu -i gpurun_out/prof_$2.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_$2_source.csv 2>&1
gzip -f gpurun_out/prof_$2_source.csv
ls -la gpurun_out
