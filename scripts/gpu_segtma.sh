#!/bin/bash
# TMA-ring fixed-segment kernel: parity (forced paths), A/B timing vs LDG
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_segtma.py tests/test_gpu_segmented.py -x -q > gpurun_out/segtma_tests.log 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/segtma_tests.log
for p in ldg tma; do
  PP_SEG_PATH=$p timeout 300 python scripts/seg_ab.py 2>&1 | sed "s/^/$p /"
done
timeout 300 python bench.py --config c4seg --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_c4seg.log 2>&1
echo "bench rc=$?"; tail -1 gpurun_out/bench_c4seg.log | cut -c1-300
