#!/usr/bin/env python3
"""Experiment: count a pinned (UVA-mapped) host buffer in
place over PCIe vs the pipelined copy path.  Needs a build whose
check_device_ptr (csrc/pp_api.cu) also accepts cudaMemoryTypeHost pointers
with a device mapping -- the shipped library rejects them."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2412_16370_b200 import _lib
from oracle import oracle as O
lib = _lib.load()
n = 1 << 30
pin = torch.empty(n, dtype=torch.uint8, pin_memory=True)
pin.copy_(torch.from_numpy(np.random.default_rng(3).integers(0, 256, n, dtype=np.uint8)))
cnt = torch.zeros(64, dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for path in ("mapped", "copy"):
    ts = []
    for _ in range(4):
        cnt.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if path == "mapped":
            _lib.check(lib.pp_count(pin.data_ptr(), n, 8, cnt.data_ptr(), sp))
            torch.cuda.synchronize()
        else:
            out = np.zeros(64, np.uint64)
            _lib.check(lib.pp_count_host(pin.data_ptr(), n, 8, out.ctypes.data))
        ts.append(time.perf_counter() - t0)
    print(path, [f"{n / t / 1e9:.1f}GB/s" for t in ts], flush=True)
if True:
    want = O.hs512(pin.numpy(), 0, n, 8, threads=16)
    cnt.zero_()
    _lib.check(lib.pp_count(pin.data_ptr(), n, 8, cnt.data_ptr(), sp))
    torch.cuda.synchronize()
    print("mapped exact:", [int(x) for x in cnt[:8].cpu()] == want)
