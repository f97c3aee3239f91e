#!/usr/bin/env python3
"""Back-to-back pp_count on an L2-resident buffer (C4's 64 MiB at offset 3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
buf = gen.generate("bernoulli", (64 << 20) + 64, 0xC4, q=655)
cnt = torch.zeros(64, dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for n, off in ((64 << 20, 3), (64 << 20, 0), (32 << 20, 0), (16 << 20, 0)):
    f = lambda: _lib.check(lib.pp_count(buf.data_ptr() + off, n, 64, cnt.data_ptr(), sp))
    for _ in range(20):
        f()
    torch.cuda.synchronize()
    torch.cuda._sleep(1000000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        f()
    b.record(); torch.cuda.synchronize()
    us = a.elapsed_time(b) / 50 * 1e3
    print(f"{os.path.basename(_lib.LIB_PATH)} {n >> 20}MiB+{off}: {us:.2f} us {n / us / 1e3:.0f} GB/s", flush=True)
