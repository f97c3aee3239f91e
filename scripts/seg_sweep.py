#!/usr/bin/env python3
"""Fixed-segment throughput by segment size (auto lanes), current PP_SEG_PATH."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
n = 1 << 30
buf = gen.generate("bernoulli", n, 0xC5, q=655)
sp = torch.cuda.current_stream().cuda_stream
path = os.environ.get("PP_SEG_PATH", "auto")
for w in (64, 8):
    for seg in (256, 1024, 2048, 4096, 8192, 16384, 65536):
        nseg = n // seg
        out = torch.zeros((nseg, w), dtype=torch.int64, device="cuda")
        f = lambda: _lib.check(lib.pp_count_fixed(buf.data_ptr(), seg, nseg, w, out.data_ptr(), 1, sp))
        for _ in range(3):
            f()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(10):
            f()
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        print(f"{path} w={w} seg={seg} us={ms*1e3:.1f} inout_GBs={(n + nseg * w * 8) / ms / 1e6:.0f}", flush=True)
        del out
