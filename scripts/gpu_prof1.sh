set -x
python __graft_entry__.py > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_segmented.py -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_seg.log 2>&1; echo pytest=$?
python scripts/prof_kernels.py --reps 3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/prof_kernels.py --reps 3 > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
python scripts/prof_kernels.py --reps 2 > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pp_ -c 6 -o gpurun_out/prof_r1 python scripts/prof_kernels.py --reps 2 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/ncu_full.log
