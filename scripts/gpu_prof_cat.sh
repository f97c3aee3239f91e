#!/bin/bash
# full ncu capture of the fused one-hot producer at w = 8/16/32/64 (+ launch list)
mkdir -p gpurun_out
P="python scripts/prof_kernels.py --reps 1 --which cat"
$P > gpurun_out/prof_cat_plain.log 2>&1; echo plain=$?
ncu --set full --clock-control none --import-source on -k regex:pp_tma_kernel -c 4 -o gpurun_out/prof_r2_cat $P > gpurun_out/ncu_cat.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_cat.log
