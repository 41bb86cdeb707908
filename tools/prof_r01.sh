# ncu captures for round 1 (run under gpurun; the plain run of each command precedes its ncu run)
P="python tools/profile_forward.py"
$P --mode forward --batch 256 > gpurun_out/pf_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_forward_b256.csv $P --mode forward --batch 256 > gpurun_out/ncu1.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_ks_modup -c 1 -o gpurun_out/prof_modup $P --mode forward --batch 256 > gpurun_out/ncu3.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_ks_ip -c 1 -o gpurun_out/prof_ip $P --mode forward --batch 256 > gpurun_out/ncu4.log 2>&1
$P --mode ntt > gpurun_out/pn_plain.log 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_ntt_batch -c 1 -o gpurun_out/prof_ntt $P --mode ntt > gpurun_out/ncu2.log 2>&1
for r in prof_modup prof_ip prof_ntt; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>&1
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>&1
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_source.csv 2>&1
done
rm -f gpurun_out/prof_ip.ncu-rep gpurun_out/prof_ntt.ncu-rep
gzip -f gpurun_out/*_source.csv
ls -la gpurun_out; du -sh gpurun_out
