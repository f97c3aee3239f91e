#!/usr/bin/env python3
"""Upper bound for a length-sorted segment order: the same length multiset
laid out in random vs descending-length order, G = 8/16/32 (1 GiB, w=64)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
sp = torch.cuda.current_stream().cuda_stream
rng = np.random.default_rng(11)
n = 1 << 30
buf = gen.generate("bernoulli", n, 0xC4, q=655)
K = 1024
cases = {
    "uni0-4K": lambda m: rng.integers(0, 4 * K // 8, m) * 8,
    "uni0-8K": lambda m: rng.integers(0, 8 * K // 8, m) * 8,
    "uni0-16K": lambda m: rng.integers(0, 16 * K // 8, m) * 8,
    "exp4K": lambda m: (rng.exponential(4 * K / 8, m).astype(np.int64)) * 8,
    "lognorm4K": lambda m: (np.exp(rng.normal(np.log(4 * K / 8), 1.0, m)).astype(np.int64)) * 8,
}
for name, mk in cases.items():
    lens0 = mk(1_200_000).astype(np.int64)
    lens0 = lens0[: np.searchsorted(np.cumsum(lens0), n)]
    for order in ("random", "sorted"):
        lens = lens0 if order == "random" else np.sort(lens0)[::-1]
        offs = np.zeros(lens.size + 1, dtype=np.int64)
        offs[1:] = np.cumsum(lens)
        d = torch.from_numpy(offs).cuda()
        nseg = lens.size
        out = torch.zeros((nseg, 64), dtype=torch.int64, device="cuda")
        row = []
        for lanes in (8, 16, 32):
            fl = 1 | (lanes << 8)
            f = lambda: _lib.check(lib.pp_count_segmented(buf.data_ptr(), d.data_ptr(), nseg, 64, out.data_ptr(), fl, sp))
            for _ in range(3):
                f()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); a.record()
            for _ in range(10):
                f()
            b.record(); torch.cuda.synchronize()
            row.append(f"G{lanes}={a.elapsed_time(b) / 10 * 1e3:.1f}")
        print(f"{name:10s} {order:6s} nseg={nseg} us: " + " ".join(row), flush=True)
        del out
