#!/usr/bin/env python3
"""Dynamic chunk order threshold: warm back-to-back and cold (L2 flushed)
single launches at 16-256 MiB (A/B builds via PP_LIB_PATH)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
label = sys.argv[1]
buf = gen.generate("uniform", 256 << 20, 0xC2)
cnt = torch.zeros(64, dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sink = torch.zeros((), dtype=torch.int64, device="cuda")
row = []
for mib in (16, 32, 64, 128, 256):
    n = mib << 20
    f = lambda: _lib.check(lib.pp_count(buf.data_ptr(), n, 8, cnt.data_ptr(), sp))
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    torch.cuda._sleep(1_000_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        f()
    b.record()
    torch.cuda.synchronize()
    warm = a.elapsed_time(b) / 50 * 1e3
    cold = 0.0
    for _ in range(10):
        flush.fill_(1)
        sink.copy_(flush.view(torch.int64).max())
        a.record(); f(); b.record()
        torch.cuda.synchronize()
        cold += a.elapsed_time(b) * 1e3 / 10
    row.append(f"{mib}MiB warm={warm:.2f} cold={cold:.2f}")
print(label, " | ".join(row))
