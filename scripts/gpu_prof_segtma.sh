#!/bin/bash
# full ncu capture of the fixed-segment TMA kernel (C4 batch, 1 GiB)
P="python scripts/prof_kernels.py --reps 2 --which seg"
$P > gpurun_out/prof_seg_plain.log 2>&1; echo plain=$?
ncu --set full --clock-control none --import-source on -k regex:pp_segtma -c 2 -o gpurun_out/prof_r1d_segtma $P > gpurun_out/ncu_segtma.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_segtma.log
