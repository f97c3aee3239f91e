#!/bin/bash
# PP_CLC=1 (chunk order by cluster launch control) vs the ticket scheduler:
# parity suites on the variant, then the bench lines of both, two passes
set -u
mkdir -p gpurun_out
V=scripts/variants/lib_clc.so
PP_LIB_PATH=$V timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_categories.py tests/test_gpu_fused.py -q -x -p no:cacheprovider --timeout 600 > gpurun_out/clc_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/clc_tests.log
B="--no-e2e --no-cpu-baseline --no-strong-c5 --no-all-configs"
for pass in 1 2; do
  for cfg in c2 c3 c4 c1 c5 c3cat; do
    for lib in default $V; do
      if [ $lib = default ]; then unset PP_LIB_PATH; else export PP_LIB_PATH=$lib; fi
      timeout 300 python bench.py --config $cfg $B 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('$cfg', '$lib', d['value'], d['unit'], 'exact', d['exact'], 'ro', d['roofline'].get('readonly_roofline_gbs') or d['roofline'].get('hbm', {}).get('readonly_roofline_gbs'))
"
    done
  done
done 2>&1 | tee gpurun_out/clc_ab.log
