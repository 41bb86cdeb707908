timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
P="python tools/profile_forward.py"
$P --mode forward --batch 256 > gpurun_out/pf_plain.log 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_ks_modup -c 1 -o gpurun_out/prof_modup $P --mode forward --batch 256 > gpurun_out/ncu3.log 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:k_ks_moddown_out -c 1 -o gpurun_out/prof_mdo $P --mode forward --batch 256 > gpurun_out/ncu4.log 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:k_bsgs_mac -c 1 -o gpurun_out/prof_mac $P --mode forward --batch 256 > gpurun_out/ncu5.log 2>&1
for r in prof_modup prof_mdo prof_mac; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>&1
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>&1
done
ncu -i gpurun_out/prof_modup.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_modup_source.csv 2>&1
gzip -f gpurun_out/*_source.csv
rm -f gpurun_out/prof_mdo.ncu-rep gpurun_out/prof_mac.ncu-rep
du -sh gpurun_out
tail -2 gpurun_out/bench_full.log gpurun_out/bench_ref.log
