#!/bin/bash
set -e
cd "$(dirname "$0")/../paper_2107_07776_b200"
OBJS=$(ls build/*.o | grep -v fast_d3.o)
for px in "$@"; do
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -DDGB_SIP_PX3=$px -c csrc/fast_d3.cu -o ../tune/fast_d3_sp$px.o &
done
wait
for px in "$@"; do nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ../tune/libdgb_sp$px.so $OBJS ../tune/fast_d3_sp$px.o; done
