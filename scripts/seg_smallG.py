#!/usr/bin/env python3
"""Fixed 0.5-4 KiB segments, 1 GiB: one lane (SWAR) vs G = 2 / 4 / 8 lanes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
n = 1 << 30
buf = gen.generate("bernoulli", n + 64, 0xC5, q=655)
off = int(os.environ.get("OFF", "0"))
sp = torch.cuda.current_stream().cuda_stream
for w in (64, 8):
    for seg in (128, 256, 512, 1024, 2048, 4096):
        nseg = n // seg
        out = torch.zeros((nseg, w), dtype=torch.int64, device="cuda")
        row = []
        for lanes in (1, 2, 4, 8):
            f = lambda: _lib.check(lib.pp_count_fixed(buf.data_ptr() + off, seg, nseg, w, out.data_ptr(), 1 | (lanes << 8), sp))
            for _ in range(3):
                f()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); a.record()
            for _ in range(10):
                f()
            b.record(); torch.cuda.synchronize()
            row.append(f"G{lanes}={a.elapsed_time(b) / 10 * 1e3:.1f}")
        print(f"w={w} seg={seg} us: " + " ".join(row), flush=True)
        del out
