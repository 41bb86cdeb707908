# usage: bash tools/prof_one_kernel.sh <kernel function name> <tag> [launch-skip]
K=$1; T=$2; SKIP=${3:-0}
P="python tools/profile_forward.py --mode forward --batch 256"
$P > gpurun_out/pf_$T.log 2>&1 || exit 1
ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base function -k "$K" --launch-skip $SKIP -c 1 -o gpurun_out/prof_$T $P > gpurun_out/ncu_$T.log 2>&1
ncu -i gpurun_out/prof_$T.ncu-rep --page raw --csv > gpurun_out/prof_${T}_raw.csv 2>&1
ncu -i gpurun_out/prof_$T.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${T}_source.csv 2>&1
gzip -f gpurun_out/prof_${T}_source.csv
rm -f gpurun_out/prof_$T.ncu-rep
