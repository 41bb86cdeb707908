for cfg in "1 0" "2 0" "2 1" "1 1"; do
  set -- $cfg
  CKKS_IPQ_BB=$1 CKKS_IP_SPLIT=$2 timeout 600 python bench.py --no-cpu-baseline --no-extras --no-e2e > gpurun_out/bench_bb$1_s$2.log 2>&1
done
