#!/bin/bash
for i in 1 2; do
timeout 300 python bench.py --config c4 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c4_$i.log 2>&1
tail -1 gpurun_out/c4_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl', d['value'], d['ms_per_step'])"
done
PP_NO_PDL=1 timeout 300 python bench.py --config c4 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c4_n.log 2>&1
tail -1 gpurun_out/c4_n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nopdl', d['value'], d['ms_per_step'])"
PP_PDL_MAX_MIB=32 timeout 300 python bench.py --config c4 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c4_m.log 2>&1
tail -1 gpurun_out/c4_m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl<32MiB', d['value'], d['ms_per_step'])"
