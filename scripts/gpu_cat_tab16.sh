#!/bin/bash
# W = 16: share of the codes whose one-hot word comes from the shared-memory table
# (PP_CAT_TAB16 of 64; variants scripts/variants/lib_h<share>.so), then the category tests on one
mkdir -p gpurun_out
for pass in 1 2; do
  for v in scripts/variants/lib_h*.so; do
    PP_LIB_PATH=$v ONEHOT_ONLY=1 timeout 200 python scripts/cat_ab.py | sed "s|^|$(basename $v .so) |"
  done
done 2>&1 | tee gpurun_out/tab16_ab.log
PP_LIB_PATH=scripts/variants/lib_h14.so timeout 600 python -m pytest tests/test_gpu_categories.py -q -x -p no:cacheprovider 2>&1 | tail -2
