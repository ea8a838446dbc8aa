#!/bin/bash
# Build libdgb variants with different momentum (K=3) CTA shapes into tune/ (C T pairs as args).
set -e
cd "$(dirname "$0")/../paper_2107_07776_b200"
OBJS=$(ls build/*.o | grep -v fast_d3.o)
for ct in "$@"; do
  C=${ct%,*}; T=${ct#*,}
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -DDGB_MOM2_C=$C -DDGB_MOM2_T=$T \
    -c csrc/fast_d3.cu -o ../tune/fast_d3_${C}_${T}.o &
done
wait
for ct in "$@"; do
  C=${ct%,*}; T=${ct#*,}
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ../tune/libdgb_${C}_${T}.so $OBJS ../tune/fast_d3_${C}_${T}.o
done
