for i in 1 2; do for K in 96 192; do
echo "cur $(HLF_VAR_SEP=1 python tools/time_kernel.py 3 3 ${K}x${K}x${K} 3)"
for l in paper_1808_10481_b200/lib/exp_*.so; do echo "$(basename $l .so) $(HLF_VAR_SEP=1 HLF_B200_LIB_OVERRIDE=$l python tools/time_kernel.py 3 3 ${K}x${K}x${K} 3)"; done
done; done
