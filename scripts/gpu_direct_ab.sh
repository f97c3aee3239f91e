#!/bin/bash
# A/B of the direct small-call path (pp_count_direct_kernel): off, and its
# size cut-offs for host bytes / device bytes (scripts/latency.py rows).
set -u
mkdir -p gpurun_out
PP_NO_DIRECT=1 python scripts/latency.py --json gpurun_out/lat_base.json > gpurun_out/lat_base.log 2>&1; echo base=$?
python scripts/latency.py --json gpurun_out/lat_direct.json > gpurun_out/lat_direct.log 2>&1; echo direct=$?
for m in 65536 131072 262144 1048576; do
  PP_DIRECT_HOST_MAX=$m PP_DIRECT_DEVICE_MAX=$m python scripts/latency.py --json gpurun_out/lat_direct_$m.json > gpurun_out/lat_direct_$m.log 2>&1; echo max$m=$?
done
