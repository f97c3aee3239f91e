#!/bin/bash
timeout 100 python scripts/l2_probe.py > gpurun_out/l2.txt 2>&1; head -1 gpurun_out/l2.txt
for s in 20 100; do
  timeout 300 python bench.py --config c4 --steps $s --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c4_$s.log 2>/dev/null
  tail -1 gpurun_out/c4_$s.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('steps', d['steps'], d['value'], d['ms_per_step'], d['roofline']['achieved'])"
done
