#!/usr/bin/env python3
"""Pinned host -> device copy bandwidth: chunk size x concurrent streams
(is the e2e path's 55 GB/s the link's limit?)."""
import time
import torch
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for nst in (1, 2, 4):
    sts = [torch.cuda.Stream() for _ in range(nst)]
    for chunk_mib in (4, 16, 32, 128):
        c = chunk_mib << 20
        def run():
            for i, off in enumerate(range(0, n, c)):
                with torch.cuda.stream(sts[i % nst]):
                    d[off:off + c].copy_(h[off:off + c], non_blocking=True)
            torch.cuda.synchronize()
        run()
        t0 = time.perf_counter()
        for _ in range(3):
            run()
        t = (time.perf_counter() - t0) / 3
        print(f"streams={nst} chunk={chunk_mib}MiB {n / t / 1e9:.1f} GB/s", flush=True)
