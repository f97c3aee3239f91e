#!/usr/bin/env python3
"""Back-to-back pp_count device time per launch at a few sizes (A/B of builds
via PP_LIB_PATH): python scripts/count_ab.py [label]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
label = sys.argv[1] if len(sys.argv) > 1 else "lib"
buf = gen.generate("uniform", 1 << 30, 0xC2)
cnt = torch.zeros(64, dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
row = []
for mib, k in ((1024, 50), (256, 100), (16, 400), (1, 1000)):
    n = mib << 20
    f = lambda: _lib.check(lib.pp_count(buf.data_ptr(), n, 8, cnt.data_ptr(), sp))
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    torch.cuda._sleep(1_000_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        f()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / k * 1e3
    row.append(f"{mib}MiB={us:.2f}us({n / us / 1e3:.0f}GB/s)")
print(label, " ".join(row))
