#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_segmented.py tests/test_gpu_segtma.py -q -x > gpurun_out/segsched_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/segsched_tests.log
for p in 1 2; do
timeout 120 python scripts/seg_ab.py | grep lanes=8 | sed 's/^/dyn /'
PP_STATIC_SCHED=1 timeout 120 python scripts/seg_ab.py | grep lanes=8 | sed 's/^/static /'
done
