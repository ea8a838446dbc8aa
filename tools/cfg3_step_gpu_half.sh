#!/bin/bash
# GPU half of the cfg3 full-step parity (tools/full_step_parity.py): the reference velocity
# (403 MB) travels in K chunks, one gpurun call per chunk (snapshot limit 512 MiB); the other
# chunks and the cfg2 files are listed in .gpurunignore for the call.  Run from the repo root
# after `python tools/full_step_parity.py cpu cfg3` has written parity_data/.
set -e
K=${1:-2}
cp .gpurunignore /tmp/gpurunignore.keep
[ -f parity_data/cfg3_step_ref_u.npy ] && python tools/full_step_parity.py split cfg3 $K
for ((i = 0; i < K; ++i)); do
  grep -v '^parity_data/$' /tmp/gpurunignore.keep > .gpurunignore
  echo "parity_data/cfg2_*" >> .gpurunignore
  for ((j = 0; j < K; ++j)); do
    [ $j != $i ] && echo "parity_data/cfg3_step_ref_u.${j}of${K}.npy" >> .gpurunignore
  done
  /usr/local/graft/bin/gpurun --timeout 1200 -- "python tools/full_step_parity.py gpu cfg3 $i/$K 2>&1 | tail -3"
done
cp /tmp/gpurunignore.keep .gpurunignore
python tools/full_step_parity.py merge cfg3 $K gpurun_out | tail -1 > profiles/cfg3_full_step_parity_r02.json
cat profiles/cfg3_full_step_parity_r02.json
