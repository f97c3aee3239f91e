#!/bin/bash
# A/B of the direct small-call path (pp_count_direct_kernel / _multi_kernel)
# on one box: the queued form (PP_NO_DIRECT=1), the shipped cut-offs, and
# wide cut-offs (PP_DIRECT_HOST_MAX / PP_DIRECT_DEVICE_MAX), two passes each
# (scripts/latency.py rows).
set -u
mkdir -p gpurun_out
for pass in 1 2; do
  PP_NO_DIRECT=1 python scripts/latency.py --json gpurun_out/lat_queued_$pass.json > gpurun_out/lat_queued_$pass.log 2>&1; echo queued$pass=$?
  python scripts/latency.py --json gpurun_out/lat_direct_$pass.json > gpurun_out/lat_direct_$pass.log 2>&1; echo direct$pass=$?
  PP_DIRECT_HOST_MAX=1048576 PP_DIRECT_DEVICE_MAX=16777216 python scripts/latency.py --json gpurun_out/lat_wide_$pass.json > gpurun_out/lat_wide_$pass.log 2>&1; echo wide$pass=$?
done
