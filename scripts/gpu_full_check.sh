#!/bin/bash
# round-end style check: smoke, the whole GPU suite, default bench + reference arm
set -u
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_default.log | cut -c1-400
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; echo ref=$?
tail -1 gpurun_out/bench_reference.log | cut -c1-300
