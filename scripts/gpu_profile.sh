# Profile evidence for profiles/: launch list of the bench command, full ncu
# capture of the hot kernels.  Each ncu command runs only after the same
# command exited 0 without ncu.
set -x
python __graft_entry__.py > /dev/null 2>&1
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-check --no-all-configs"
$B > gpurun_out/prof_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $B > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu_launch=$?
P="python scripts/prof_kernels.py --reps 2"
$P > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pp_ -c 10 -o gpurun_out/prof_r2 $P > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
