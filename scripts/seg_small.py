#!/usr/bin/env python3
"""Many short arrays in one segmented launch (C4's short lengths, batched):
device time per launch and per array, fixed-size segments at byte offset 3."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
sp = torch.cuda.current_stream().cuda_stream
buf = gen.generate("bernoulli", (1 << 30) + 64, 0xC4, q=655)
for words in [int(x) for x in os.environ.get("WORDS", "1,3,17,255,512,8192").split(",")]:
    seg = 8 * words
    nseg = min(1 << 20, (1 << 30) // seg)
    for w in (64, 8):
        out = torch.zeros((nseg, w), dtype=torch.int64, device="cuda")
        for lanes in (1, 8):
            f = lambda: _lib.check(lib.pp_count_fixed(buf.data_ptr() + 3, seg, nseg, w, out.data_ptr(),
                                                      1 | (lanes << 8), sp))
            for _ in range(3):
                f()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); a.record()
            for _ in range(10):
                f()
            b.record(); torch.cuda.synchronize()
            us = a.elapsed_time(b) / 10 * 1e3
            print(f"words={words} nseg={nseg} w={w} lanes={lanes} us={us:.1f} ns_per_array={us * 1e3 / nseg:.2f} "
                  f"in_GBs={seg * nseg / us / 1e3:.0f} inout_GBs={(seg + 8 * w) * nseg / us / 1e3:.0f}", flush=True)
        del out
