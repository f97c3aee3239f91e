#!/bin/bash
# Ticketed launches: trigger the successor once tickets reach the last
# PP_TRIGGER_TAIL chunks per CTA (0 = after the CTA's last load)
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["config"]["workload"][:24], d["value"], d["ms_per_step"], d["exact"], r.get("readonly_roofline_gbs") or r.get("hbm",{}).get("readonly_roofline_gbs"))'
for pass in 1 2 3; do
for t in 0 2 4 8 16; do
  for cfg in c2 c3; do
    PP_TRIGGER_TAIL=$t timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-strong-c5 --no-all-configs | python -c "$J" | sed "s/^/tail$t $cfg /"
  done
done
done
