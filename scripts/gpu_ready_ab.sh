#!/bin/bash
# PP_COUNT_INPUT_READY: exactness, then bench lines with / without the flag
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_segmented.py -q -x -p no:cacheprovider > gpurun_out/ready_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/ready_tests.log
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"][:28], d["value"], d["ms_per_step"], d["exact"], d.get("launch","")[:20])'
for pass in 1 2; do
for cfg in c1 c4 c2; do
  timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-strong-c5 | python -c "$J" | sed "s/^/ready $cfg /"
  timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-strong-c5 --no-input-ready | python -c "$J" | sed "s/^/plain $cfg /"
done
done
