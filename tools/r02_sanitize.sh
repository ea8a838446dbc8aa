#!/bin/bash
# compute-sanitizer evidence for the hot kernels (SPEC.md:279
# "face loops race-free"): a clean plain run first, then racecheck (shared-memory
# hazards), synccheck (illegal __syncwarp / barrier use) and memcheck, restricted to
# this library's kernels (namespace dgb).  Summaries -> gpurun_out/sanitize_*.txt
mkdir -p gpurun_out
python tools/sanitize_cases.py > gpurun_out/sanitize_plain.txt 2>&1 || exit 1
for tool in racecheck synccheck memcheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --kernel-name regex:dgb --print-limit 50 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$tool.txt
done
