#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_categories.py -q -x > gpurun_out/cat_v2_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/cat_v2_tests.log
for pass in 1 2; do
ONEHOT_ONLY=1 timeout 200 python scripts/cat_ab.py | sed 's/^/v2 /'
ONEHOT_ONLY=1 PP_LIB_PATH=scripts/variants/lib_catv1.so timeout 200 python scripts/cat_ab.py | sed 's/^/v1 /'
done
