#!/bin/bash
# A/B the fixed-segment TMA kernel variants (scripts/variants/lib_*.so), 2 passes
for pass in 1 2; do
for v in scripts/variants/lib_*.so; do
  PP_LIB_PATH=$v timeout 120 python scripts/seg_ab.py 2>&1 | grep lanes=8
done
done
