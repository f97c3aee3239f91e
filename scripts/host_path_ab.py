#!/usr/bin/env python3
"""pospopcnt(bytes) throughput by size (pageable host input), current env."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_16370_b200 as pp
rng = np.random.default_rng(1)
tag = os.environ.get("TAG", "")
for mib in (1, 2, 4, 8, 16, 32, 64, 256):
    data = rng.integers(0, 256, mib << 20, dtype=np.uint8).tobytes()
    for _ in range(3):
        pp.pospopcnt(data, 8)
    k = max(5, min(50, 2048 // mib))
    t0 = time.perf_counter()
    for _ in range(k):
        pp.pospopcnt(data, 8)
    dt = (time.perf_counter() - t0) / k
    print(f"{tag} {mib}MiB {dt * 1e6:.0f}us {(mib << 20) / dt / 1e9:.1f}GB/s", flush=True)
