#!/bin/bash
# end-of-round evidence in one call: smoke, GPU suite, default bench +
# reference arm, every-config bench lines, launch list + ncu of the hot kernels
set -u
mkdir -p gpurun_out
bash scripts/gpu_final.sh
bash scripts/gpu_bench_all.sh > gpurun_out/bench_all.log 2>&1; echo bench_all=$?
