# memcheck of the edge-case driver (one compute-sanitizer tool per call), after
# the same command exited 0 without the sanitizer.
set -x
python __graft_entry__.py > /dev/null 2>&1
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 600 python scripts/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1; echo plain=$?
tail -2 gpurun_out/sanitize_plain.log
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/memcheck.log 2>&1; echo memcheck=$?
tail -6 gpurun_out/memcheck.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "all_widths or graph" > gpurun_out/pytest_new.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_new.log
