#!/usr/bin/env python3
"""Ragged (CSR) segmented throughput, static vs dynamic order via PP_STATIC_SCHED."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
sp = torch.cuda.current_stream().cuda_stream
rng = np.random.default_rng(5)
n = 1 << 30
buf = gen.generate("bernoulli", n, 0xC4, q=655)
tag = "static" if os.environ.get("PP_STATIC_SCHED") else "dynamic"
cases = {
    "uniform0-16K": lambda: rng.integers(0, 2048, 200_000) * 8,
    "skewed": lambda: np.where(rng.random(400_000) < 0.9, 64, 64 * 1024 // 4),
}
for name, mk in cases.items():
    lens = mk().astype(np.int64)
    lens = lens[: np.searchsorted(np.cumsum(lens), n)]
    offs = np.zeros(lens.size + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens)
    d = torch.from_numpy(offs).cuda()
    nseg = lens.size
    for lanes, extra in ((8, 0), (32, 0), (8, _lib.PP_SEG_HYBRID), (16, _lib.PP_SEG_HYBRID), (0, 0)):
        out = torch.zeros((nseg, 64), dtype=torch.int64, device="cuda")
        f = lambda: _lib.check(lib.pp_count_segmented(buf.data_ptr(), d.data_ptr(), nseg, 64, out.data_ptr(), 1 | (lanes << 8) | extra, sp))
        for _ in range(3):
            f()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(10):
            f()
        b.record(); torch.cuda.synchronize()
        us = a.elapsed_time(b) / 10 * 1e3
        tot = int(offs[-1]) + nseg * 512
        print(f"{tag} {name} nseg={nseg} lanes={lanes}{'+hybrid' if extra else ''} us={us:.1f} inout_GBs={tot / us / 1e3:.0f}", flush=True)
