#!/bin/bash
# static lead chunks before the first ticket (PP_STATIC_LEAD 3 vs 1)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_categories.py tests/test_gpu_fused.py -q -x > gpurun_out/lead_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/lead_tests.log
for pass in 1 2 3; do
python scripts/count_ab.py lead3
PP_LIB_PATH=scripts/variants/lib_lead1.so python scripts/count_ab.py lead1
done
PP_LIB_PATH=scripts/variants/lib_tl.so python scripts/timeline.py
python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline | cut -c1-200
