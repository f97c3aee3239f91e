#!/bin/bash
# W = 32: share of the one-hot words loaded from the shared-memory table
# (PP_CAT_TAB32 of 32, 3-stage ring kept; variants scripts/variants/lib_u<share>.so)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_categories.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/tab32_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/tab32_tests.log
for pass in 1 2; do
  ONEHOT_ONLY=1 timeout 200 python scripts/cat_ab.py | sed "s/^/default /"
  for v in scripts/variants/lib_u*.so; do
    PP_LIB_PATH=$v ONEHOT_ONLY=1 timeout 200 python scripts/cat_ab.py | sed "s|^|$(basename $v .so) |"
  done
done 2>&1 | tee gpurun_out/tab32_ab.log
