# one ncu --set full capture per kernel regex (first matching launch of one profiled forward, B=256)
P="python tools/profile_forward.py"
$P --mode forward --batch 256 > gpurun_out/pf_plain.log 2>&1 || exit 1
for spec in "$@"; do
  re=${spec%%:*}; tag=${spec##*:}
  ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$re -c 1 -o gpurun_out/prof_$tag $P --mode forward --batch 256 > gpurun_out/ncu_$tag.log 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_source.csv 2>&1
  gzip -f gpurun_out/prof_${tag}_source.csv
  rm -f gpurun_out/prof_$tag.ncu-rep
done
ls -la gpurun_out
