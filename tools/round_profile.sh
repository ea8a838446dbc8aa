#!/bin/bash
# Bench line + ncu launch list + one full capture of the two hot kernels (run on the GPU box).
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --steps 2 --warmup 1 --no-step --no-cpu > /dev/null 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-step --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_momentum_axis|k_sip_axis' -c 2 \
  -o gpurun_out/full_r1 -f python bench.py --steps 2 --warmup 1 --no-step --no-cpu > gpurun_out/ncu_full.log 2>&1
