#!/usr/bin/env python3
"""Ragged (CSR) segments: which G (lanes per segment) wins, against the count
mean and the byte-weighted mean (sum L^2 / sum L) of the lengths."""
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
    "fixed4K": lambda m: np.full(m, 4 * K),
    "fixed8K": lambda m: np.full(m, 8 * K),
    "uni0-4K": lambda m: rng.integers(0, 4 * K // 8, m) * 8,
    "uni0-8K": lambda m: rng.integers(0, 8 * K // 8, m) * 8,
    "uni0-16K": lambda m: rng.integers(0, 16 * K // 8, m) * 8,
    "uni0-32K": lambda m: rng.integers(0, 32 * K // 8, m) * 8,
    "uni4K-12K": lambda m: rng.integers(4 * K // 8, 12 * K // 8, m) * 8,
    "exp2K": lambda m: (rng.exponential(2 * K / 8, m).astype(np.int64)) * 8,
    "exp4K": lambda m: (rng.exponential(4 * K / 8, m).astype(np.int64)) * 8,
    "exp8K": lambda m: (rng.exponential(8 * K / 8, m).astype(np.int64)) * 8,
    "lognorm4K": lambda m: (np.exp(rng.normal(np.log(4 * K / 8), 1.0, m)).astype(np.int64)) * 8,
}
w = int(os.environ.get("W", "64"))
TS = [int(x) for x in os.environ.get("TS", "0").split(",")]
for name, mk in cases.items():
    lens = mk(1_200_000).astype(np.int64)
    lens = lens[: np.searchsorted(np.cumsum(lens), n)]
    offs = np.zeros(lens.size + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens)
    d = torch.from_numpy(offs).cuda()
    nseg = lens.size
    mean = lens.mean()
    bmean = (lens.astype(np.float64) ** 2).sum() / max(lens.sum(), 1)
    out = torch.zeros((nseg, w), dtype=torch.int64, device="cuda")
    row = []
    for lanes, T in [(g, t) for g in (8, 16, 32) for t in TS]:
        fl = 1 | (lanes << 8) | (T << _lib.PP_SEG_BATCH_SHIFT)
        f = lambda: _lib.check(lib.pp_count_segmented(buf.data_ptr(), d.data_ptr(), nseg, w, out.data_ptr(), fl, sp))
        for _ in range(3):
            f()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(10):
            f()
        b.record(); torch.cuda.synchronize()
        row.append(f"G{lanes}T{T or 'a'}={a.elapsed_time(b) / 10 * 1e3:.1f}")
    from paper_2412_16370_b200 import segmented as S
    auto = S._shape(nseg, int(lens.max()), S._byte_mean(lens), False)[0]
    print(f"w={w} {name:10s} autoG={auto:2d} nseg={nseg:7d} mean={mean/K:6.2f}K bmean={bmean/K:6.2f}K us: " + " ".join(row), flush=True)
    del out
