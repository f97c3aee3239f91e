#!/usr/bin/env python3
"""Fused categories throughput when every u8 code is valid for the width (uniform in [0, w)),
beside the C3 draws (Zipf over 32 categories) scripts/cat_ab.py uses at every width."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16370_b200 import _lib
lib = _lib.load()
n = 1 << 30
cnt = torch.zeros(64, dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
g = torch.Generator(device="cuda"); g.manual_seed(5)
for w in (8, 16, 32, 64):
    codes = torch.randint(0, w, (n,), dtype=torch.uint8, device="cuda", generator=g)
    f = lambda: _lib.check(lib.pp_count_categories(codes.data_ptr(), n, 1, w, cnt.data_ptr(), sp))
    for _ in range(3):
        f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(10):
        f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"uniform codes in [0,{w}): w{w} = {n / ms / 1e6:.0f} G codes/s", flush=True)
    del codes
