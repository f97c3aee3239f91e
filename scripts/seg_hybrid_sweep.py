#!/usr/bin/env python3
"""Bimodal CSR lengths: G-lane kernel alone vs the hybrid split (tiny arrays
one lane each), per G; prints the fractions the auto rule could key on."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
sp = torch.cuda.current_stream().cuda_stream
rng = np.random.default_rng(12)
n = 1 << 30
buf = gen.generate("bernoulli", n, 0xC4, q=655)
K = 1024
def bimodal(p, a, b):
    return lambda m: np.where(rng.random(m) < p, a, b)
cases = {
    "90%64B/16K": bimodal(0.9, 64, 16 * K),
    "90%64B/4K": bimodal(0.9, 64, 4 * K),
    "70%256B/4K": bimodal(0.7, 256, 4 * K),
    "50%128B/8K": bimodal(0.5, 128, 8 * K),
    "50%512B/2K": bimodal(0.5, 512, 2 * K),
    "97%32B/64K": bimodal(0.97, 32, 64 * K),
    "80%0-512/0-32K": lambda m: np.where(rng.random(m) < 0.8, rng.integers(0, 64, m) * 8,
                                         rng.integers(0, 4 * K, m) * 8),
}
w = 64
for name, mk in cases.items():
    lens = mk(4_000_000).astype(np.int64)
    lens = lens[: np.searchsorted(np.cumsum(lens), n)]
    offs = np.zeros(lens.size + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens)
    d = torch.from_numpy(offs).cuda()
    nseg = lens.size
    short = lens <= 512
    fs, fb = short.mean(), lens[short].sum() / lens.sum()
    long_ = lens[~short].astype(np.float64)
    lbm = (long_ ** 2).sum() / max(long_.sum(), 1)
    bm = (lens.astype(np.float64) ** 2).sum() / lens.sum()
    out = torch.zeros((nseg, w), dtype=torch.int64, device="cuda")
    row = []
    for lanes in (1, 8, 16, 32):
        for hyb in ((0,) if lanes == 1 else (0, 1)):
            fl = 1 | (lanes << 8) | (_lib.PP_SEG_HYBRID if hyb else 0)
            f = lambda: _lib.check(lib.pp_count_segmented(buf.data_ptr(), d.data_ptr(), nseg, w, out.data_ptr(), fl, sp))
            for _ in range(3):
                f()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); a.record()
            for _ in range(10):
                f()
            b.record(); torch.cuda.synchronize()
            row.append(f"G{lanes}{'h' if hyb else ''}={a.elapsed_time(b) / 10 * 1e3:.1f}")
    print(f"{name:15s} nseg={nseg:7d} short_frac={fs:.2f} short_bytes={fb:.3f} bmean={bm/K:.1f}K long_bmean={lbm/K:.1f}K us: " + " ".join(row), flush=True)
    del out
