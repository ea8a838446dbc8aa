#!/bin/bash
# Build libdgb variants of the generic 3D k=4 kernels with (threads, smem budget KB) pairs.
set -e
cd "$(dirname "$0")/../paper_2107_07776_b200"
OBJS=$(ls build/*.o | grep -v ops_d3_k4.o)
for tk in "$@"; do
  T=${tk%,*}; KB=${tk#*,}
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -DDGB_GMOM_T=$T -DDGB_GMOM_KB=$KB \
    -c csrc/ops_d3_k4.cu -o ../tune/ops_d3_k4_${T}_${KB}.o &
done
wait
for tk in "$@"; do
  T=${tk%,*}; KB=${tk#*,}
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ../tune/libdgb_g${T}_${KB}.so $OBJS ../tune/ops_d3_k4_${T}_${KB}.o
done
