#!/usr/bin/env python3
"""Single launches after an L2 flush, bracketed by CUDA events: the
measurement floor (16 B) vs 2 MiB / 64 MiB counts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
buf = gen.generate("uniform", 64 << 20, 0xC1)
cnt = torch.zeros(64, dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sink = torch.zeros((), dtype=torch.int64, device="cuda")
tiny = torch.zeros(16, dtype=torch.float32, device="cuda")
for label, f in (("torch add_ (16 floats)", lambda: tiny.add_(1.0)),
                 ("pp_count 16 B", lambda: _lib.check(lib.pp_count(buf.data_ptr(), 16, 8, cnt.data_ptr(), sp))),
                 ("pp_count 2 MiB", lambda: _lib.check(lib.pp_count(buf.data_ptr(), 2 << 20, 16, cnt.data_ptr(), sp))),
                 ("pp_count 64 MiB", lambda: _lib.check(lib.pp_count(buf.data_ptr(), 64 << 20, 64, cnt.data_ptr(), sp)))):
    tot, n = 0.0, 20
    for i in range(n + 3):
        flush.fill_(1)
        sink.copy_(flush.view(torch.int64).max())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record()
        torch.cuda.synchronize()
        if i >= 3:
            tot += a.elapsed_time(b) * 1e3
    print(f"{label:24s} {tot / n:.2f} us")
