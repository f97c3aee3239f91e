set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_segmented.py -m gpu -q -x -p no:cacheprovider --timeout 600 > gpurun_out/pytest_seg.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_seg.log
timeout 300 python scripts/seg_ab.py
