#!/usr/bin/env python3
"""C4 batch and other fixed / ragged shapes, µs per launch (A/B via PP_LIB_PATH)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
sp = torch.cuda.current_stream().cuda_stream
n = 1 << 30
buf = gen.generate("bernoulli", n + 64, 0xC5, q=655)
out = torch.empty(((1 << 20) * 64,), dtype=torch.int64, device="cuda")
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
for seg, off in ((4096, 0), (1024, 3), (8, 3), (16384, 0), (8192, 0), (8192, 3)):
    nseg = min(1 << 20, n // seg)
    row.append(f"fixed{seg}@{off}={t(lambda: _lib.check(lib.pp_count_fixed(buf.data_ptr() + off, seg, nseg, 64, out.data_ptr(), 1, sp))):.1f}")
rng = np.random.default_rng(1)
lens = rng.integers(0, 1024, 200_000) * 8
offs = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)])).cuda()
row.append(f"ragged0-8K={t(lambda: _lib.check(lib.pp_count_segmented(buf.data_ptr(), offs.data_ptr(), lens.size, 64, out.data_ptr(), 1, sp))):.1f}")
print(sys.argv[1], " ".join(row))
