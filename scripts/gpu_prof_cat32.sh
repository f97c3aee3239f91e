#!/bin/bash
# ncu --set full of the w=32 categories kernel: small-code fast path vs base build
mkdir -p gpurun_out
P="python scripts/prof_kernels.py --reps 1 --which cat"
$P > gpurun_out/prof_cat_plain.log 2>&1; echo plain=$?
ncu --set full --clock-control none --import-source on -k regex:pp_tma_kernel --launch-skip 2 -c 1 -o gpurun_out/prof_cat32_small $P > gpurun_out/ncu_cat32.log 2>&1; echo ncu=$?
PP_LIB_PATH=scripts/variants/lib_nosmall.so ncu --set full --clock-control none --import-source on -k regex:pp_tma_kernel --launch-skip 2 -c 1 -o gpurun_out/prof_cat32_base $P > gpurun_out/ncu_cat32b.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_cat32*.log
