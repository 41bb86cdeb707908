# builds the variants of tools/lab/ntt_lab.cu into tools/lab/bin/
set -e
cd "$(dirname "$0")"
mkdir -p bin
rm -f bin/*
I=../../paper_2205_11935_b200/csrc
build() { name=$1; shift; nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -I$I -I../../include "$@" -DLAB_NAME="\"$name\"" ntt_lab.cu -o bin/$name & }
for st in 0 1 2; do
build c14_st$st -DLAB_MINB=2 -DNTTC_ST_DEFAULT=$st
build c14_r_st$st -DLAB_MINB=2 -DLAB_R -DNTTC_ST_DEFAULT=$st
build c13_st$st -DLAB_LOGN=13 -DLAB_MINB=2 -DNTTC_ST_DEFAULT=$st
build c12_st$st -DLAB_LOGN=12 -DLAB_MINB=4 -DNTTC_ST_DEFAULT=$st
done
wait
ls bin
