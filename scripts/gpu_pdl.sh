set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do
for pdl in 0 1; do
  if [ $pdl = 0 ]; then export PP_NO_PDL=1; else unset PP_NO_PDL; fi
  python bench.py --steps 50 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$pdl', d['value'], d['roofline']['readonly_roofline_gbs'], d['per_width_gbs'], d['exact'])"
done; done
for pdl in 0 1; do
  if [ $pdl = 0 ]; then export PP_NO_PDL=1; else unset PP_NO_PDL; fi
  python bench.py --config c1 --steps 200 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 pdl=$pdl', d['value'], d['ms_per_step'], d['exact'])"
  python bench.py --config c3cat --steps 20 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3cat pdl=$pdl', d['value'], d['exact'])"
done
