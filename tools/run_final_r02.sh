# r02 final evidence: GPU suite, smoke, bench (both arms), launch list of one B = 256 forward chunk, ncu --set full of
# the top kernels of the forward and of the cfg2 batch NTT (cluster schedule).  Outputs under gpurun_out/final/.
set -x
O=gpurun_out/final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
(timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -15) > $O/pytest_gpu_all.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python bench.py > $O/bench_full.log 2>&1; echo "bench rc=$?" >> $O/bench_full.log
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_reference.log 2>&1; echo "rc=$?" >> $O/bench_reference.log
P="python tools/profile_forward.py --mode forward --batch 256"
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_forward_b256.csv $P > $O/ncu_launches.log 2>&1
# name:tag:launch-skip (function base names; skip picks the dense1 instance of each)
for spec in "k_ks_ip_mma3:ipmma3:0" "k_ks_modup_c:modup2:3" "k_bsgs_mac_mma:macmma:0" "k_ks_digits:digits:1" "k_ks_ip_giant_multi:ipgiant:0"; do
  IFS=: read k tag skip <<< "$spec"
  ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base function -k "$k" --launch-skip $skip -c 1 -o $O/prof_$tag $P > $O/ncu_$tag.log 2>&1
  ncu -i $O/prof_$tag.ncu-rep --page raw --csv > $O/prof_${tag}_raw.csv 2>&1
  ncu -i $O/prof_$tag.ncu-rep --page source --csv --print-source sass > $O/prof_${tag}_source.csv 2>&1
  gzip -f $O/prof_${tag}_source.csv
  rm -f $O/prof_$tag.ncu-rep
done
P2="python tools/profile_forward.py --mode ntt"
ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base function -k "k_ntt_batch_c" -c 2 -o $O/prof_nttbatch $P2 > $O/ncu_nttbatch.log 2>&1
ncu -i $O/prof_nttbatch.ncu-rep --page raw --csv > $O/prof_nttbatch_raw.csv 2>&1
ncu -i $O/prof_nttbatch.ncu-rep --page source --csv --print-source sass > $O/prof_nttbatch_source.csv 2>&1
gzip -f $O/prof_nttbatch_source.csv
rm -f $O/prof_nttbatch.ncu-rep
cuobjdump -sass paper_2205_11935_b200/_build/libckks_b200.so | grep -E "UBLKCP|UTMALDG|UTCIMMA|UTCHMMA|SYNCS|DMMA" | awk '{print $2}' | sort | uniq -c | sort -rn | head -30 > $O/sass_mnemonics.txt
