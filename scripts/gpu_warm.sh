#!/bin/bash
# headline stability vs warm-up length (cold-start effects on the first timed region)
for w in 5 5 50 5 200 5; do
python bench.py --steps 20 --warmup $w --no-e2e --no-cpu-baseline --no-check | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('warmup', $w, d['value'], d['roofline']['readonly_roofline_gbs'], d['per_width_gbs'])"
done
