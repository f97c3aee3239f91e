#!/bin/bash
# A/B of the direct small-call path (pp_count_direct_kernel) on one box: the
# queued form (PP_NO_DIRECT=1) and the shipped one, two passes each
# (scripts/latency.py rows); PP_DIRECT_HOST_MAX / PP_DIRECT_DEVICE_MAX move
# the size cut-offs (256 KiB shipped).
set -u
mkdir -p gpurun_out
for pass in 1 2; do
  PP_NO_DIRECT=1 python scripts/latency.py --json gpurun_out/lat_queued_$pass.json > gpurun_out/lat_queued_$pass.log 2>&1; echo queued$pass=$?
  python scripts/latency.py --json gpurun_out/lat_direct_$pass.json > gpurun_out/lat_direct_$pass.log 2>&1; echo direct$pass=$?
done
