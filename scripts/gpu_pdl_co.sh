#!/bin/bash
# PDL at every size with the max-shared carveout (co-resident next grid)
for pass in 1 2; do
PP_NO_PDL=1 timeout 120 python scripts/pdl_sweep.py
PP_PDL_MAX_MIB=4096 timeout 120 python scripts/pdl_sweep.py
PP_PDL_MAX_MIB=4096 PP_LIB_PATH=scripts/variants/lib_co.so timeout 120 python scripts/pdl_sweep.py | sed 's/^/co-/'
PP_NO_PDL=1 PP_LIB_PATH=scripts/variants/lib_co.so timeout 120 python scripts/pdl_sweep.py | sed 's/^/co-/'
done
