#!/usr/bin/env python3
"""Per-CTA %globaltimer timeline of one counting launch (PP_TIMELINE build):
PP_LIB_PATH=scripts/variants/lib_tl.so python scripts/timeline.py [MiB]."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
n = int(sys.argv[1]) << 20 if len(sys.argv) > 1 else 1 << 30
buf = gen.generate("uniform", n, 0xC2)
cnt = torch.zeros(64, dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for _ in range(20):
    _lib.check(lib.pp_count(buf.data_ptr(), n, 8, cnt.data_ptr(), sp))
torch.cuda.synchronize()
# one launch after a spin so it runs alone, and one in a back-to-back pair
tl = np.zeros((1024, 8), dtype=np.uint64)
f = lib.pp_debug_timeline
f.argtypes = [ctypes.c_void_p]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sink = torch.zeros((), dtype=torch.int64, device="cuda")
for label, k in (("alone", 1), ("back-to-back (last of 10)", 10), ("cold (L2 flushed)", 1)):
    if label.startswith("cold"):
        flush.fill_(1)
        sink.copy_(flush.view(torch.int64).max())
    else:
        torch.cuda._sleep(1000000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        _lib.check(lib.pp_count(buf.data_ptr(), n, 8, cnt.data_ptr(), sp))
    b.record()
    torch.cuda.synchronize()
    assert f(tl.ctypes.data) == 0
    g = int(min(148, (n + 32767) // 32768))
    t = tl[:g].astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3  # us
    names = ["entry", "1st copy issued", "1st stage consumed", "last copy issued",
             "last chunk consumed", "epilogue start", "end"]
    print(f"== {label}: {n >> 20} MiB, {g} CTAs, events {a.elapsed_time(b) / k * 1e3:.2f} us/launch")
    for i, nm in enumerate(names):
        c = rel[:, i]
        print(f"  {nm:22s} min {c.min():8.2f}  median {np.median(c):8.2f}  max {c.max():8.2f} us")
