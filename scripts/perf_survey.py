#!/usr/bin/env python3
"""One table of device times across entry points and shapes (anomaly hunt).

  python scripts/perf_survey.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_16370_b200 as pp  # noqa: E402
from paper_2412_16370_b200 import _lib, gen  # noqa: E402

MIB = 1 << 20


def timed(f, reps=10, warm=3):
    for _ in range(warm):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    lib = _lib.load()
    sp = torch.cuda.current_stream().cuda_stream
    buf = gen.generate("uniform", (1 << 30) + 64, 0xC2)
    cnt = torch.zeros(64, dtype=torch.int64, device="cuda")
    rows = []

    def add(name, us, nbytes=None):
        rows.append((name, us, None if nbytes is None else nbytes / us / 1e3))

    for n in (1 * MIB, 16 * MIB, 256 * MIB, 1 << 30):
        for off in (0, 5):
            add(f"pp_count w=16 {n >> 20} MiB +{off}",
                timed(lambda: _lib.check(lib.pp_count(buf.data_ptr() + off, n, 16,
                                                      cnt.data_ptr(), sp))), n)
    add("pp_count_frame 1 GiB", timed(lambda: _lib.check(
        lib.pp_count_frame(buf.data_ptr(), 1 << 30, cnt.data_ptr(), sp))), 1 << 30)
    add("pp_readonly_sum 1 GiB", timed(lambda: _lib.check(
        lib.pp_readonly_sum(buf.data_ptr(), 1 << 30, cnt.data_ptr(), sp))), 1 << 30)
    tg = (__import__("ctypes").c_void_p * 2)(cnt.data_ptr(), cnt.data_ptr() + 512)
    add("pp_count_multi 1 GiB (2 local targets)", timed(lambda: _lib.check(
        lib.pp_count_multi(buf.data_ptr(), 1 << 30, 8, tg, 2, sp))), 1 << 30)
    for cb, dt in ((1, torch.uint8), (2, torch.int16), (4, torch.int32)):
        n = (1 << 30) // cb
        codes = buf[: n * cb].view(dt) if cb > 1 else buf[:n]
        codes = (codes.to(torch.int64) % 40).to(dt) if cb > 1 else codes.clone() % 40
        for w in (8, 32, 64):
            add(f"categories {dt} w={w} ({n >> 20} Mi codes)", timed(lambda: _lib.check(
                lib.pp_count_categories(codes.data_ptr(), n, cb, w, cnt.data_ptr(), sp)), reps=5),
                n * cb)
        del codes
    out = torch.empty((1 << 20) * 64, dtype=torch.int64, device="cuda")
    for seg in (8, 64, 512, 1024, 4096, 65536):
        nseg = min(1 << 20, (1 << 30) // seg)
        for off in (0, 3):
            add(f"pp_count_fixed w=64 {nseg} x {seg} B +{off}", timed(lambda: _lib.check(
                lib.pp_count_fixed(buf.data_ptr() + off, seg, nseg, 64, out.data_ptr(), 1, sp))),
                nseg * seg)
    rng = np.random.default_rng(1)
    lens = rng.integers(0, 4096, 200000) // 8 * 8
    offs = np.zeros(lens.size + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens)
    doffs = torch.from_numpy(offs).cuda()
    add("pospopcnt_segmented ragged 0-4 KiB (Python API, host offsets)",
        timed(lambda: pp.pospopcnt_segmented(buf[: int(offs[-1])], offs, 64)), int(offs[-1]))
    add("pospopcnt_segmented ragged 0-4 KiB (device offsets, no validation)",
        timed(lambda: pp.pospopcnt_segmented(buf[: int(offs[-1])], doffs, 64, validate=False)),
        int(offs[-1]))
    arrays = [buf[int(offs[i]):int(offs[i + 1])] for i in range(2000)]
    add("pospopcnt_batch 2000 separate views", timed(lambda: pp.pospopcnt_batch(arrays, 64)),
        int(offs[2000]))
    add("pospopcnt_all_widths 256 MiB", timed(lambda: pp.pospopcnt_all_widths(
        buf[: 256 * MIB]), reps=5), 256 * MIB)
    for name, us, gbs in rows:
        print(f"{name:60s} {us:10.2f} us" + (f" {gbs:9.1f} GB/s" if gbs else ""), flush=True)


if __name__ == "__main__":
    main()
