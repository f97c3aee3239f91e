#!/usr/bin/env python3
"""Ragged CSR segments: plain segmented count vs SegmentPlan (length-sorted
processing order), per G (1 GiB, w=64, us per launch; plan built once)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2412_16370_b200 as pp
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
    "uni0-32K": lambda m: rng.integers(0, 32 * K // 8, m) * 8,
    "exp2K": lambda m: (rng.exponential(2 * K / 8, m).astype(np.int64)) * 8,
    "exp4K": lambda m: (rng.exponential(4 * K / 8, m).astype(np.int64)) * 8,
    "exp8K": lambda m: (rng.exponential(8 * K / 8, m).astype(np.int64)) * 8,
    "lognorm4K": lambda m: (np.exp(rng.normal(np.log(4 * K / 8), 1.0, m)).astype(np.int64)) * 8,
    "90%64B/16K": lambda m: np.where(rng.random(m) < 0.9, 64, 16 * K),
}
def t_us(f):
    for _ in range(3):
        f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(10):
        f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / 10 * 1e3
view = pp.InputView(buf, 0, n)
for name, mk in cases.items():
    lens = mk(4_000_000).astype(np.int64)
    lens = lens[: np.searchsorted(np.cumsum(lens), n)]
    offs = np.zeros(lens.size + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens)
    d = torch.from_numpy(offs).cuda()
    nseg = lens.size
    out = torch.zeros((nseg, 64), dtype=torch.int64, device="cuda")
    row = []
    auto = pp.SegmentPlan(offs, device="cuda")
    row.append(f"plain-auto(G{auto.lanes}{'h' if auto.hybrid else ''})="
               f"{t_us(lambda: pp.pospopcnt_segmented(view, d, 64, out=out, accumulate=False, validate=False, lanes=auto.lanes, hybrid=auto.hybrid)):.1f}")
    row.append(f"plan-auto={t_us(lambda: auto.count(view, 64, out=out, accumulate=False)):.1f}")
    for g in (8, 16, 32):
        pl = pp.SegmentPlan(offs, device="cuda", lanes=g, hybrid=False)
        fl = 1 | (g << 8)
        row.append(f"G{g}:plain={t_us(lambda: _lib.check(lib.pp_count_segmented(buf.data_ptr(), d.data_ptr(), nseg, 64, out.data_ptr(), fl, sp))):.1f}"
                   f"/plan={t_us(lambda: pl.count(view, 64, out=out, accumulate=False)):.1f}")
    print(f"{name:11s} nseg={nseg:7d} " + " ".join(row), flush=True)
    del out
