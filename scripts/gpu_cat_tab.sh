#!/bin/bash
# One-hot words from per-lane shared-memory tables for a share of the codes
# (PP_CAT_TAB64 of 16 / PP_CAT_TAB32 of 32, pp_count.cu KShape): exactness of
# the default build, then throughput of every variant built into
# scripts/variants/lib_t*.so (two interleaved passes)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_categories.py -q -x -p no:cacheprovider > gpurun_out/tab_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/tab_tests.log
for pass in 1 2; do
  ONEHOT_ONLY=1 timeout 200 python scripts/cat_ab.py | sed "s/^/default /"
  for v in scripts/variants/lib_t*.so; do
    PP_LIB_PATH=$v ONEHOT_ONLY=1 timeout 200 python scripts/cat_ab.py | sed "s|^|$(basename $v .so) |"
  done
done 2>&1 | tee gpurun_out/tab_ab.log
