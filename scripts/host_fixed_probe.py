#!/usr/bin/env python3
"""Where the per-call cost of pp_count_host on pageable inputs goes: the C entry
point alone vs the Python API, by size; PP_HOST_STAGE_MIN / PP_HOST_STAGE_CHUNK /
PP_HOST_COPY_THREADS from the environment."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_16370_b200 as pp
from paper_2412_16370_b200 import _lib
lib = _lib.load()
rng = np.random.default_rng(1)
out = np.zeros(64, dtype=np.uint64)
tag = os.environ.get("TAG", "")
for mib in [float(x) for x in os.environ.get("SIZES", "2,4,8,16,32,64,128,256,1024").split(",")]:
    nb = int(mib * (1 << 20))
    arr = rng.integers(0, 256, nb, dtype=np.uint8)
    data = arr.tobytes()
    k = max(3, min(200, int(2048 // mib)))
    f_c = lambda: _lib.check(lib.pp_count_host(arr.ctypes.data, arr.size, 8, out.ctypes.data))
    f_py = lambda: pp.pospopcnt(data, 8)
    res = []
    for f in (f_c, f_py):
        for _ in range(3):
            f()
        ts = []
        for _ in range(k):
            t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
        ts.sort()
        res.append((ts[len(ts) // 2], ts[0]))
    print(f"{tag} {mib:9.4f} MiB  C median {res[0][0]*1e6:8.0f} us (min {res[0][1]*1e6:8.0f}) {nb/res[0][0]/1e9:6.1f} GB/s"
          f" | py median {res[1][0]*1e6:8.0f} us {nb/res[1][0]/1e9:6.1f} GB/s", flush=True)
