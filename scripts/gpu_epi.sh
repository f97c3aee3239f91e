#!/bin/bash
# per-warp frame rows vs shared u64 atomics in the counting kernel's epilogue
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_categories.py -q -x > gpurun_out/epi_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/epi_tests.log
for pass in 1 2 3; do
python scripts/count_ab.py rows
PP_LIB_PATH=scripts/variants/lib_epi0.so python scripts/count_ab.py atom
done
PP_LIB_PATH=scripts/variants/lib_tl.so python scripts/timeline.py
PP_LIB_PATH=scripts/variants/lib_tl_epi0.so python scripts/timeline.py
