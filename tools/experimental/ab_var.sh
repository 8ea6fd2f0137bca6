#!/bin/bash
# A/B of the var2d kernel: current lib vs lib/exp_*.so; usage: ab_var.sh "m ..." reps
ms=${1:-"3"}; reps=${2:-2}
for i in $(seq $reps); do for m in $ms; do
  echo "cur  $(python tools/experimental/var2d_time.py $m)"
  for l in paper_1808_10481_b200/lib/exp_*.so; do
    [ -e "$l" ] || continue
    echo "$(basename $l .so) $(HLF_B200_LIB_OVERRIDE=$l python tools/experimental/var2d_time.py $m)"
  done
done; done
