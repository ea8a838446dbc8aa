#!/bin/bash
# Build libdgb variants with different cells-per-CTA caps of k_momentum_qp into tune/ (caps as args);
# time them on the GPU box with: DGB_LIB=tune/libdgb_mqp<c>.so python tools/cfg_apply_timing.py cfg4
set -e
mkdir -p "$(dirname "$0")/../tune"
cd "$(dirname "$0")/../paper_2107_07776_b200"
OBJS=$(ls build/*.o | grep -v fast_d3.o)
for c in "$@"; do
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -DDGB_MQP_CMAX=$c \
    -c csrc/fast_d3.cu -o ../tune/fast_d3_mqp$c.o &
done
wait
for c in "$@"; do
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ../tune/libdgb_mqp$c.so $OBJS ../tune/fast_d3_mqp$c.o
done
