#!/usr/bin/env python3
"""A/B timing of segmented-kernel variants: PP_LIB_PATH=<so> python scripts/seg_ab.py."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
n = 1 << 30
buf = gen.generate("bernoulli", n, 0xC5, q=655)
out = torch.zeros((n // 4096, 64), dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for L, P in ((8, 0), (16, 0), (32, 0)):
    f = lambda: _lib.check(lib.pp_count_fixed(buf.data_ptr(), 4096, n // 4096, 64, out.data_ptr(), 1 | (L << 8) | P, sp))
    for _ in range(5):
        f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(20):
        f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"{os.path.basename(_lib.LIB_PATH)} lanes={L} us={ms*1e3:.1f} inout_GBs={(n + n // 4096 * 512) / ms / 1e6:.0f}")
