#!/bin/bash
# Static lead chunks per CTA before the first ticket (PP_STATIC_LEAD; the
# default is the ring depth), exactness first (scheduler, golden, checked build)
mkdir -p gpurun_out
LEADS=${LEADS:-"3 1 2"}
if [ -z "${NO_TESTS:-}" ]; then
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_checked.py tests/test_gpu_categories.py -q -x -p no:cacheprovider > gpurun_out/lead_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/lead_tests.log
fi
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"][:24], d["value"], d["ms_per_step"], d["exact"], d["roofline"]["readonly_roofline_gbs"] if "readonly_roofline_gbs" in d["roofline"] else d["roofline"].get("hbm",{}).get("readonly_roofline_gbs"))'
for pass in 1 2 3; do
for lead in $LEADS; do
for cfg in ${CFGS:-c2 c3}; do
  PP_STATIC_LEAD=$lead timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-strong-c5 --no-all-configs | python -c "$J" | sed "s/^/lead$lead $cfg /"
done
done
done
