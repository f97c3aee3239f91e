#!/bin/bash
# L2 bulk prefetch in pp_seg_kernel: PP_SEG_PF = 1 (default build) vs 0 vs 2
timeout 900 python -m pytest tests/test_gpu_segmented.py tests/test_gpu_edges.py -q -x > gpurun_out/segpf_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/segpf_tests.log
for pass in 1 2; do
for v in 1 0 2; do
L=""; [ $v != 1 ] && L="PP_LIB_PATH=scripts/variants/lib_segpf$v.so"
env $L timeout 300 python scripts/seg_ragged.py | sed "s/^/pf$v /"
env $L OFF=3 timeout 300 python scripts/seg_smallG.py | sed "s/^/pf$v /"
done
done
