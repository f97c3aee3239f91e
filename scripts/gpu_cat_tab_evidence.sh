#!/bin/bash
# after the W=64 table path: categories + checked-build + fuzz tests, then the
# ALU / LSU pipe counts of the fused producer at every width (cat_alu.csv)
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_categories.py tests/test_gpu_checked.py tests/test_gpu_fuzz.py -q -p no:cacheprovider --timeout 900 > gpurun_out/tab_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/tab_pytest.log
P="python scripts/prof_kernels.py --reps 1 --which cat"
$P > gpurun_out/alu_plain.log 2>&1 && \
ncu --metrics sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_lsu.sum,smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:pp_tma_kernel --csv --log-file gpurun_out/cat_alu.csv $P > gpurun_out/ncu_alu.log 2>&1; echo ncu_alu=$?
{ for dt in uint8 int16 int32; do CAT_DTYPE=$dt ONEHOT_ONLY=1 timeout 300 python scripts/cat_ab.py; done; timeout 300 python scripts/cat_range_probe.py; } | tee gpurun_out/cat_ab_final.log
timeout 300 python bench.py --config c3cat --no-e2e --no-cpu-baseline > gpurun_out/bench_c3cat.log 2>&1; echo c3cat=$?
