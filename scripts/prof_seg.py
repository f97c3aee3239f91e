#!/usr/bin/env python3
"""ncu driver: segmented kernels (TMA and LDG paths, G=8) on 262,144 x 4 KiB."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
n = 1 << 30
buf = gen.generate("bernoulli", n, 0xC5, q=655)
out = torch.zeros((n // 4096, 64), dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for P in (0,):
    for _ in range(2):
        _lib.check(lib.pp_count_fixed(buf.data_ptr(), 4096, n // 4096, 64, out.data_ptr(), 1 | (8 << 8) | P, sp))
torch.cuda.synchronize()
print("ok")
