O=gpurun_out/final
P="python tools/profile_forward.py --mode forward --batch 256"
for spec in "k_ks_modup_c:modup2:3" "k_ks_ip_giant_multi:ipgiant:0"; do
  IFS=: read k tag skip <<< "$spec"
  ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base function -k "$k" --launch-skip $skip -c 1 -o $O/prof_$tag $P > $O/ncu_$tag.log 2>&1
  ncu -i $O/prof_$tag.ncu-rep --page raw --csv > $O/prof_${tag}_raw.csv 2>&1
  ncu -i $O/prof_$tag.ncu-rep --page source --csv --print-source sass > $O/prof_${tag}_source.csv 2>&1
  gzip -f $O/prof_${tag}_source.csv
  rm -f $O/prof_$tag.ncu-rep
done
