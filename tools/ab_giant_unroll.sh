# A/B of the giant-step IP batch unroll / occupancy (libraries prebuilt under _ab/)
B=paper_2205_11935_b200/_build/libckks_b200.so
cp $B _ab/lib_orig.so
for v in u4m4 u8m4 u4m5 u6m4 u2m4 u4m4; do
  cp _ab/lib_$v.so $B
  timeout 300 python bench.py --no-cpu-baseline --no-extras --no-e2e > gpurun_out/bench_g_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_g_$v.log').read().strip().splitlines()[-1]);print('$v',d['value'],d['kernel_shares']['k_ks_ip_giant']['ms_per_step'])" >> gpurun_out/ab_giant.txt 2>&1
done
cp _ab/lib_orig.so $B
