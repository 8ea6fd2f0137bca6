#!/bin/bash
# Energy per step of the stage ablation builds (tools/build_exp.sh NAME -DHLF_EXP_*):
# every launch runs at the board's power cap, so time x power attributes the
# step's energy to its stages.  usage: tools/ablation_power.sh > out.jsonl
echo "{\"lib\": \"full\", \"r\": $(python tools/launch_power.py 3 512x512x256 step)}"
for l in paper_1808_10481_b200/lib/exp_*.so; do
  n=$(basename $l .so)
  extra=""
  [ "$n" = "exp_notgt" ] && extra="HLF_NO_TMA_T=1"
  echo "{\"lib\": \"$n\", \"r\": $(env $extra HLF_B200_LIB_OVERRIDE=$l python tools/launch_power.py 3 512x512x256 step)}"
done
