#!/bin/bash
# TMA ring depth of the counting kernel (dynamic order + PDL), 1 GiB and 256 MiB
for pass in 1 2; do
for n in 2 3 4 5 6; do
  PP_LIB_PATH=scripts/variants/lib_st$n.so timeout 120 python scripts/pdl_sweep.py | sed "s/^/st$n /"
done
done
