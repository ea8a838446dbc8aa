#!/bin/bash
# Build libdgb variants of the Gram-Schmidt dot pass into tune/: args "minblocks:gridcap" pairs;
# time with DGB_LIB=tune/libdgb_gs<m>_<c>.so CFG=3 DGB_GMRES_PROF=1 python tools/step_timing.py
set -e
mkdir -p "$(dirname "$0")/../tune"
cd "$(dirname "$0")/../paper_2107_07776_b200"
OBJS=$(ls build/*.o | grep -v blas.o)
for v in "$@"; do
  m=${v%%:*}; c=${v##*:}
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -DDGB_GSD_MINB=$m -DDGB_GS_CAP=$c \
    -c csrc/blas.cu -o ../tune/blas_gs${m}_$c.o &
done
wait
for v in "$@"; do
  m=${v%%:*}; c=${v##*:}
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ../tune/libdgb_gs${m}_$c.so $OBJS ../tune/blas_gs${m}_$c.o
done
