#!/bin/bash
# A/B device timing: current lib vs paper_1808_10481_b200/lib/exp_*.so variants.
# usage: tools/ab.sh "d m K" reps
args=${1:-"3 3 512x512x256"}; reps=${2:-2}
for i in $(seq $reps); do
  echo "cur  $(python tools/time_kernel.py $args 10)"
  for l in paper_1808_10481_b200/lib/exp_*.so; do
    [ -e "$l" ] || continue
    echo "$(basename $l .so) $(HLF_B200_LIB_OVERRIDE=$l python tools/time_kernel.py $args 10)"
  done
done
