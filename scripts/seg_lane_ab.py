#!/usr/bin/env python3
"""One-lane kernel shapes, µs per launch (A/B via PP_LIB_PATH)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
sp = torch.cuda.current_stream().cuda_stream
n = 1 << 30
buf = gen.generate("bernoulli", n + 64, 0xC5, q=655)
out = torch.empty(((1 << 21) * 64,), dtype=torch.int64, device="cuda")
def t(f, k=10):
    for _ in range(3):
        f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(k):
        f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / k * 1e3
row = []
for seg, off, w in ((8, 3, 64), (64, 0, 64), (256, 0, 64), (512, 3, 64), (256, 0, 8), (512, 0, 8)):
    nseg = min(1 << 21, n // seg)
    fl = 1 | (1 << 8)
    row.append(f"{seg}B@{off}w{w}={t(lambda: _lib.check(lib.pp_count_fixed(buf.data_ptr() + off, seg, nseg, w, out.data_ptr(), fl, sp))):.1f}")
print(sys.argv[1], " ".join(row))
