# Full GPU check: build, smoke, gpu tests, default bench line.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1; echo build=$?
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo benchref=$?
tail -5 gpurun_out/pytest_gpu.log
cat gpurun_out/bench.log gpurun_out/bench_ref.log
