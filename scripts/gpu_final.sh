#!/bin/bash
# round-end evidence: smoke, GPU suite, default bench + reference arm, then
# the launch list of the bench command and a full ncu capture of the hot kernels
set -u
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; echo ref=$?
bash scripts/gpu_profile.sh > gpurun_out/profile.log 2>&1; echo profile=$?
tail -3 gpurun_out/profile.log
