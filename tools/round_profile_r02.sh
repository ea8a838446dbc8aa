#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun): GPU tests, bench line, reference arm,
# ncu launch list of the bench, full captures of the cfg3 and cfg4 hot kernels.
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-step --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_momentum_axis|k_sip_cell|k_sip_axis' -c 2 \
  -o gpurun_out/full_r02 -f python bench.py --steps 2 --warmup 1 --no-step --no-cpu > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_momentum_qp|k_sip_qp' -c 2 \
  -o gpurun_out/cfg4_r02b -f python tools/prof_cfg4_mom.py > gpurun_out/ncu4.log 2>&1
