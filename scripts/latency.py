#!/usr/bin/env python3
"""Per-call latency across input sizes: device time per launch (CUDA events
around back-to-back launches) and the host cost of each API layer.

  python scripts/latency.py [--json out.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    import torch
    import paper_2412_16370_b200 as pp
    from paper_2412_16370_b200 import _lib, gen
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    big = gen.generate("uniform", 64 << 20, 0xC1, device=dev)
    cnt = torch.zeros(64, dtype=torch.int64, device=dev)
    rows = []
    for n in (8, 64, 1024, 4096, 16384, 32768, 65536, 131072, 262144, 524288, 1 << 20, 2 << 20, 4 << 20,
              16 << 20,
              64 << 20):
        w = 16
        ptr = big.data_ptr() + 3 if n < (64 << 20) else big.data_ptr()
        nn = n if n < (64 << 20) else n
        k = 200 if n <= (2 << 20) else 50
        for _ in range(10):
            _lib.check(lib.pp_count(ptr, nn, w, cnt.data_ptr(), sp))
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        t0 = time.perf_counter()
        for _ in range(k):
            _lib.check(lib.pp_count(ptr, nn, w, cnt.data_ptr(), sp))
        t_cabi = (time.perf_counter() - t0) / k
        b.record(st)
        torch.cuda.synchronize()
        dev_us = a.elapsed_time(b) / k * 1e3
        view = pp.InputView(big, 3, nn) if n < (64 << 20) else big
        pp.pospopcnt(view, w, counters=cnt)  # first calls set up per-thread buffers
        pp.pospopcnt(view, w)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k):
            pp.pospopcnt(view, w, counters=cnt)
        torch.cuda.synchronize()
        t_api_dev = (time.perf_counter() - t0) / k
        t0 = time.perf_counter()
        kk = min(k, 50)
        for _ in range(kk):
            pp.pospopcnt(view, w)
        t_api_list = (time.perf_counter() - t0) / kk
        host = big[:nn].cpu().numpy().tobytes()
        pp.pospopcnt(host, w)  # first use of a path allocates its pinned buffers
        t0 = time.perf_counter()
        for _ in range(kk):
            pp.pospopcnt(host, w)
        t_api_bytes = (time.perf_counter() - t0) / kk
        # the synchronous C-ABI calls without the Python layer: device bytes ->
        # host counters (pp_count_sync), host bytes -> host counters (pp_count_host)
        import ctypes
        import numpy as np
        hc = np.zeros(64, dtype=np.uint64)
        hb = np.frombuffer(host, dtype=np.uint8)
        for _ in range(3):
            _lib.check(lib.pp_count_sync(ptr, nn, w, hc.ctypes.data, sp))
            _lib.check(lib.pp_count_host(hb.ctypes.data, nn, w, hc.ctypes.data))
        t0 = time.perf_counter()
        for _ in range(kk):
            _lib.check(lib.pp_count_sync(ptr, nn, w, hc.ctypes.data, sp))
        t_sync = (time.perf_counter() - t0) / kk
        t0 = time.perf_counter()
        for _ in range(kk):
            _lib.check(lib.pp_count_host(hb.ctypes.data, nn, w, hc.ctypes.data))
        t_host = (time.perf_counter() - t0) / kk
        row = {"bytes": n, "device_us_per_launch": round(dev_us, 2),
               "c_abi_call_us": round(t_cabi * 1e6, 2),
               "c_abi_sync_us": round(t_sync * 1e6, 2),
               "c_abi_host_us": round(t_host * 1e6, 2),
               "api_device_counters_us": round(t_api_dev * 1e6, 2),
               "api_list_counters_us": round(t_api_list * 1e6, 2),
               "api_host_bytes_us": round(t_api_bytes * 1e6, 2),
               "device_GBs": round(n / dev_us / 1e3, 1)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
