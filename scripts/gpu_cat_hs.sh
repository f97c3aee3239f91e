#!/bin/bash
# A/B of the categories counters: chunk-batched CatCounter (default) vs the
# per-group Counter (lib_cat_old, built before the change), and consumer
# warps per CTA (16 default, 15, 12).  Exactness first.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_categories.py -q -x -p no:cacheprovider > gpurun_out/cat_hs_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/cat_hs_tests.log
for v in lib_cat_ncw15 lib_cat_ncw12; do
PP_LIB_PATH=scripts/variants/$v.so timeout 900 python -m pytest tests/test_gpu_categories.py -q -x -p no:cacheprovider > gpurun_out/cat_hs_tests_$v.log 2>&1; echo tests_$v=$?; tail -1 gpurun_out/cat_hs_tests_$v.log
done
for pass in 1 2; do
for v in default lib_cat_old lib_cat_ncw15 lib_cat_ncw12; do
  if [ $v = default ]; then L=""; else L=scripts/variants/$v.so; fi
  PP_LIB_PATH=$L ONEHOT_ONLY=1 timeout 200 python scripts/cat_ab.py | sed "s/^/$v /"
done
done
