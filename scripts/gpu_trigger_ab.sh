#!/bin/bash
# Dependent-launch trigger at kernel start (default) vs after the CTA's last
# load (PP_LATE_TRIGGER=1); ticketed (default) vs static chunk order
# (PP_DYN_MIN_CHUNKS=huge).  Every config rotates over >= 3 input copies.
mkdir -p gpurun_out
if [ -z "${NO_TESTS:-}" ]; then
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_checked.py tests/test_gpu_categories.py tests/test_gpu_fused.py tests/test_gpu_segmented.py -q -x -p no:cacheprovider > gpurun_out/trig_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/trig_tests.log
fi
J='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["config"]["workload"][:24], d["value"], d["ms_per_step"], d["exact"], r.get("readonly_roofline_gbs") or r.get("hbm",{}).get("readonly_roofline_gbs"))'
for pass in 1 2; do
for v in early late early_static; do
  E=""
  case $v in late) E="PP_LATE_TRIGGER=1";; early_static) E="PP_DYN_MIN_CHUNKS=999999999";; esac
  for cfg in ${CFGS:-c2 c3 c4 c1 c3cat}; do
    env $E timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-strong-c5 --no-all-configs | python -c "$J" | sed "s/^/$v $cfg /"
  done
done
done
