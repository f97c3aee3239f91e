#!/bin/bash
# W=32 small-code path byte extraction: mul.hi (FMA pipe, default) vs plain
# shifts (ALU) vs no small path; exactness of each variant first
mkdir -p gpurun_out
for v in default lib_cat_nosmall lib_cat_shr; do
  if [ $v = default ]; then L=""; else L=scripts/variants/$v.so; fi
  PP_LIB_PATH=$L timeout 600 python -m pytest tests/test_gpu_categories.py -q -x -p no:cacheprovider > gpurun_out/cat_ab2_$v.log 2>&1; echo tests_$v=$?; tail -1 gpurun_out/cat_ab2_$v.log
done
for pass in 1 2; do
for v in default lib_cat_nosmall lib_cat_shr; do
  if [ $v = default ]; then L=""; else L=scripts/variants/$v.so; fi
  PP_LIB_PATH=$L ONEHOT_ONLY=1 timeout 200 python scripts/cat_ab.py | sed "s/^/$v /"
done
done
