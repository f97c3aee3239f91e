#!/bin/bash
# A/B of the W=16/32 small-code fast path (PP_CAT_SMALL) + the categories tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_categories.py -q -x > gpurun_out/cat_small_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/cat_small_tests.log
for pass in 1 2; do
ONEHOT_ONLY=1 timeout 200 python scripts/cat_ab.py | sed 's/^/small /'
ONEHOT_ONLY=1 PP_LIB_PATH=scripts/variants/lib_nosmall.so timeout 200 python scripts/cat_ab.py | sed 's/^/base  /'
done
