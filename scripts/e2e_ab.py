#!/usr/bin/env python3
"""pp_count_host from pinned memory, 1 GiB: GB/s (A/B via PP_LIB_PATH)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_16370_b200 as pp
n = 1 << 30
pinned = torch.empty(n, dtype=torch.uint8, pin_memory=True)
pinned.fill_(0x5A)
pp.pospopcnt(pinned, 8)
best = []
for r in range(3):
    t0 = time.perf_counter()
    for _ in range(5):
        pp.pospopcnt(pinned, 8)
    best.append(5 * n / (time.perf_counter() - t0) / 1e9)
print(sys.argv[1], " ".join(f"{x:.2f}" for x in best))
