set -x
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv
lscpu | grep -E "Model name|^CPU\(s\)|Flags" | cut -c1-150
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-min-time 3 > gpurun_out/bench_tma.log 2>&1; echo bench=$?
PP_LOAD_PATH=ldg timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_ldg.log 2>&1; echo benchldg=$?
tail -3 gpurun_out/*.log
