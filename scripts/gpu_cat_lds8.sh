#!/bin/bash
# u8 codes one byte per lane from shared memory (PP_CAT_LDS8, default since
# round 2) -- exactness of the default build, then throughput vs a variant
mkdir -p gpurun_out
V=${V:-lib_cat_lds8}
timeout 900 python -m pytest tests/test_gpu_categories.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/lds8_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/lds8_tests.log
for pass in 1 2; do
  ONEHOT_ONLY=1 timeout 200 python scripts/cat_ab.py | sed "s/^/default /"
  PP_LIB_PATH=scripts/variants/$V.so ONEHOT_ONLY=1 timeout 200 python scripts/cat_ab.py | sed "s/^/$V /"
done
