#!/bin/bash
# ncu of the ragged LDG segmented kernel with and without the L2 evict-first load hint
mkdir -p gpurun_out
python scripts/prof_ragged.py > gpurun_out/prof_ragged_plain.log 2>&1; echo plain=$?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_write.sum,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio
ncu --metrics $M --clock-control none -k regex:pp_seg_kernel -c 2 --csv python scripts/prof_ragged.py > gpurun_out/ncu_ragged_hint.csv 2>&1; echo hint=$?
PP_LIB_PATH=scripts/variants/lib_ldg0.so ncu --metrics $M --clock-control none -k regex:pp_seg_kernel -c 2 --csv python scripts/prof_ragged.py > gpurun_out/ncu_ragged_nohint.csv 2>&1; echo nohint=$?
