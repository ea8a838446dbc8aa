#!/bin/bash
# Build libdgb variants that differ only in fast_d3.cu compile flags, into tune/:
#   tools/ab_build.sh name "-DFLAG=1 ..." [name "flags" ...]
set -e
cd "$(dirname "$0")/../paper_2107_07776_b200"
mkdir -p ../tune
OBJS=$(ls build/*.o | grep -v fast_d3.o)
args=("$@")
for ((i = 0; i < ${#args[@]}; i += 2)); do
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC ${args[i+1]} \
    -c csrc/fast_d3.cu -o ../tune/fast_d3_${args[i]}.o &
done
wait
for ((i = 0; i < ${#args[@]}; i += 2)); do
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ../tune/libdgb_${args[i]}.so $OBJS ../tune/fast_d3_${args[i]}.o
done
