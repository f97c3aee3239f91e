#!/bin/bash
# consumer-warp / stage sweep of the fused one-hot producer (u8 codes)
for pass in 1 2; do
ONEHOT_ONLY=1 timeout 200 python scripts/cat_ab.py | sed 's/^/16x3 /'
for v in 12x3 20x2 24x2; do
ONEHOT_ONLY=1 PP_LIB_PATH=scripts/variants/lib_cat$v.so timeout 200 python scripts/cat_ab.py | sed "s/^/$v /"
done
done
