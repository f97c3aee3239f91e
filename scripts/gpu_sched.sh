#!/bin/bash
# dynamic vs static chunk scheduling of the TMA kernels
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_categories.py tests/test_gpu_golden.py tests/test_gpu_fused.py -q -x > gpurun_out/sched_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/sched_tests.log
for pass in 1 2; do
timeout 120 python scripts/pdl_sweep.py | sed 's/^/dyn-/'
PP_STATIC_SCHED=1 timeout 120 python scripts/pdl_sweep.py | sed 's/^/static-/'
done
for pass in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b_dyn.log 2>&1; tail -1 gpurun_out/b_dyn.log | cut -c1-120
PP_STATIC_SCHED=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b_static.log 2>&1; tail -1 gpurun_out/b_static.log | cut -c1-120
done
timeout 300 python bench.py --config c4seg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-120
