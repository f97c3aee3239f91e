#!/bin/bash
# Round-2 evidence in one call: ALU instruction counts of the fused producer
# (profiles/ncu_alu.json), every-config bench lines, the launch list of the
# default bench command and a full ncu capture of the hot kernels.
set -u
mkdir -p gpurun_out
python __graft_entry__.py > /dev/null 2>&1
P="python scripts/prof_kernels.py --reps 1 --which cat"
$P > gpurun_out/alu_plain.log 2>&1 && \
ncu --metrics sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:pp_tma_kernel --csv --log-file gpurun_out/cat_alu.csv $P > gpurun_out/ncu_alu.log 2>&1; echo ncu_alu=$?
bash scripts/gpu_bench_all.sh > gpurun_out/bench_all.log 2>&1; echo bench_all=$?
tail -3 gpurun_out/bench_all.log
bash scripts/gpu_profile.sh > gpurun_out/profile.log 2>&1; echo profile=$?
tail -3 gpurun_out/profile.log
