#!/usr/bin/env python3
"""Fused categories (u8 codes): TMA one-hot expansion vs smem histogram, per width."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
n = 1 << 30
codes = gen.generate("codes8", n, 0xC3)
dt = os.environ.get("CAT_DTYPE", "uint8")
if dt != "uint8":  # the same draws as 2- / 4-byte codes (n codes, 2n / 4n bytes)
    codes = codes.to(getattr(torch, dt))
cb = codes.element_size()
cnt = torch.zeros(64, dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for smem in (False, True) if not os.environ.get("ONEHOT_ONLY") else (False,):
    if smem:
        os.environ["PP_CAT_PATH"] = "smem"
    else:
        os.environ["PP_CAT_PATH"] = "onehot"
    row = []
    for w in (8, 16, 32, 64):
        f = lambda: _lib.check(lib.pp_count_categories(codes.data_ptr(), n, cb, w, cnt.data_ptr(), sp))
        for _ in range(3):
            f()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(10):
            f()
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        row.append(f"w{w}={n * cb / ms / 1e6:.0f}GB/s({n / ms / 1e6:.0f}Gcodes/s)")
    print(dt, "smem-hist" if smem else "tma-onehot", " ".join(row))
