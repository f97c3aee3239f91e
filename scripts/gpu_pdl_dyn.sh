#!/bin/bash
# with dynamic scheduling: does PDL now help at 1 GiB?
for pass in 1 2; do
timeout 120 python scripts/pdl_sweep.py | sed 's/^/default-/'
PP_PDL_MAX_MIB=4096 timeout 120 python scripts/pdl_sweep.py | sed 's/^/pdlall-/'
done
PP_PDL_MAX_MIB=4096 PP_LIB_PATH=scripts/variants/lib_tl.so timeout 200 python scripts/timeline.py 2>&1 | tail -8
