#!/usr/bin/env python3
"""Pageable bytes -> pospopcnt throughput (staged pinned pipeline)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_16370_b200 as pp
rng = np.random.default_rng(0)
out = []
for n in (16 << 20, 64 << 20, 256 << 20, 1 << 30):
    b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
    pp.pospopcnt(b, 8)
    reps = 5 if n < (1 << 30) else 3
    t = time.perf_counter()
    for _ in range(reps):
        pp.pospopcnt(b, 8)
    dt = (time.perf_counter() - t) / reps
    out.append(f"{n >> 20}MiB={n / dt / 1e9:.1f}")
print(os.environ.get("PP_HOST_COPY_THREADS"), os.environ.get("PP_HOST_STAGE_CHUNK"), " ".join(out))
