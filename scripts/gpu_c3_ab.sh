#!/bin/bash
# C3 (4 GiB one-hot, w=32) with the session-start build vs the current one
for pass in 1 2 3; do
python bench.py --config c3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-check | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new', d['value'], d['ms_per_step'])"
PP_LIB_PATH=scripts/variants/lib_old.so python bench.py --config c3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-check | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old', d['value'], d['ms_per_step'])"
done
