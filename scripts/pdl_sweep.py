#!/usr/bin/env python3
"""pp_count back-to-back throughput vs size (run with and without PP_NO_PDL)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
buf = gen.generate("uniform", 1 << 30, 0xC2)
cnt = torch.zeros(64, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream(); sp = st.cuda_stream
row = []
for n in (1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20, 1 << 30):
    k = max(20, min(2000, (8 << 30) // n))
    f = lambda: _lib.check(lib.pp_count(buf.data_ptr(), n, 8, cnt.data_ptr(), sp))
    for _ in range(10):
        f()
    torch.cuda.synchronize()
    torch.cuda._sleep(2000000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(k):
        f()
    b.record(st); torch.cuda.synchronize()
    us = a.elapsed_time(b) / k * 1e3
    row.append(f"{n >> 20}MiB:{us:.2f}us/{n / us / 1e3:.0f}GB/s")
print("pdl" if not os.environ.get("PP_NO_PDL") else "nopdl", " ".join(row))
