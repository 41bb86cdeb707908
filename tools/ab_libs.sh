# A/B of prebuilt library variants: bash tools/ab_libs.sh v1 v2 ...  (each _ab/lib_<v>.so, built by hand with
# the variant's -D flags); one short bench per variant, per-kernel ms of the four top kernels to gpurun_out/ab.txt
B=paper_2205_11935_b200/_build/libckks_b200.so
cp $B _ab/lib_orig.so
for v in "$@"; do
  cp _ab/lib_$v.so $B
  timeout 300 python bench.py --no-cpu-baseline --no-extras --no-e2e > gpurun_out/bench_ab_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_ab_$v.log').read().strip().splitlines()[-1]);k=d['kernel_shares'];print('$v',d['value'],{n:k[n]['ms_per_step'] for n in ['k_ks_ip_mma','k_ks_modup','k_bsgs_mac_mma','k_ks_ip_giant']})" >> gpurun_out/ab.txt 2>&1
done
cp _ab/lib_orig.so $B
