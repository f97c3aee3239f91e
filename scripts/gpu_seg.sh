set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_segmented.py tests/test_gpu_golden.py -m gpu -q -p no:cacheprovider --timeout 600 -x > gpurun_out/pytest_seg.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_seg.log
for L in 8 16 32; do python - <<PY >> gpurun_out/seg_timing.log 2>&1
import torch, sys
sys.path.insert(0,'.')
from paper_2412_16370_b200 import _lib, gen
lib=_lib.load(); n=1<<30
buf=gen.generate("bernoulli", n, 0xC5, q=655); out=torch.zeros((n//4096,64),dtype=torch.int64,device="cuda")
sp=torch.cuda.current_stream().cuda_stream
f=lambda: _lib.check(lib.pp_count_fixed(buf.data_ptr(),4096,n//4096,64,out.data_ptr(),1|($L<<8),sp))
for _ in range(5): f()
a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); a.record()
for _ in range(20): f()
b.record(); torch.cuda.synchronize(); ms=a.elapsed_time(b)/20
print("lanes=$L us=%.1f in_GBs=%.0f inout_GBs=%.0f"%(ms*1e3, n/ms/1e6, (n+n//4096*512)/ms/1e6))
PY
done
cat gpurun_out/seg_timing.log
