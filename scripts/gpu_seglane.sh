#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_segmented.py tests/test_gpu_segtma.py -x -q > gpurun_out/seglane_tests.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/seglane_tests.log
timeout 600 python scripts/seg_small.py
