set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_categories.py -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_cat.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_cat.log
PP_CAT_PATH=onehot timeout 900 python -m pytest tests/test_gpu_categories.py -m gpu -q -p no:cacheprovider --timeout 600 -k "random or c3" > gpurun_out/pytest_cat3.log 2>&1; echo pytest_onehot=$?
tail -2 gpurun_out/pytest_cat3.log
timeout 300 python scripts/cat_ab.py
