"""Performance floors: generous bounds (about 60-70 % of the round-1
measurements in profiles/) that catch gross regressions of a shape or a
dispatch rule -- e.g. the batched-ticket change that once made 1023 arrays
of 64 KiB 5x slower, or the hybrid test that cost the one-lane kernel 40 %.
Device time from CUDA events around back-to-back launches."""

import pytest

pytestmark = pytest.mark.gpu

MIB = 1 << 20


def _us_per_call(torch, f, reps=20, warm=3):
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


def test_perf_floors(cuda):
    torch, pp = cuda
    from paper_2412_16370_b200 import _lib, gen
    lib = _lib.load()
    sp = torch.cuda.current_stream().cuda_stream
    buf = gen.generate("uniform", (1 << 30) + 64, 0xC2)
    cnt = torch.zeros(64, dtype=torch.int64, device="cuda")
    out = torch.empty((1 << 20) * 64, dtype=torch.int64, device="cuda")
    checks = []

    def count(n, off=0, w=8):
        return lambda: _lib.check(lib.pp_count(buf.data_ptr() + off, n, w, cnt.data_ptr(), sp))

    def fixed(seg, nseg, off, w=64):
        return lambda: _lib.check(lib.pp_count_fixed(buf.data_ptr() + off, seg, nseg, w,
                                                     out.data_ptr(), _lib.PP_SEG_OVERWRITE, sp))

    # (name, callable, bytes for a GB/s floor or None, floor GB/s, ceiling us)
    checks.append(("C2 1 GiB w=8", count(1 << 30), 1 << 30, 5000, None))
    checks.append(("C4 batch 262144 x 4 KiB", fixed(4096, 262144, 0), None, None, 260))
    checks.append(("1M x 8 B arrays", fixed(8, 1 << 20, 3), None, None, 200))
    checks.append(("1M x 1 KiB arrays, offset 3", fixed(1024, 1 << 20, 3), None, None, 700))
    checks.append(("1023 x 64 KiB arrays, offset 3", fixed(65536, 1023, 3), None, None, 45))
    checks.append(("16384 x 64 KiB arrays", fixed(65536, 16384, 0), None, None, 260))
    bad = []
    for name, f, nbytes, floor, ceil_us in checks:
        us = _us_per_call(torch, f)
        if nbytes is not None and nbytes / us / 1e3 < floor:
            bad.append(f"{name}: {nbytes / us / 1e3:.0f} GB/s < {floor}")
        if ceil_us is not None and us > ceil_us:
            bad.append(f"{name}: {us:.1f} us > {ceil_us}")
    assert not bad, bad


def test_perf_floor_ragged_ticket_batching(cuda):
    """CSR segments at G = 16 / 32 draw scheduler tickets per group: 1 GiB of
    4 KiB segments once took 592 us at G = 32 (one atomic per segment on one
    counter); the batched tickets bring it to ~200 us."""
    import numpy as np
    torch, pp = cuda
    from paper_2412_16370_b200 import _lib, gen
    lib = _lib.load()
    sp = torch.cuda.current_stream().cuda_stream
    n = 1 << 30
    buf = gen.generate("bernoulli", n, 0xC4, q=655)
    offs = torch.arange(0, n + 1, 4096, dtype=torch.int64, device="cuda")
    nseg = offs.numel() - 1
    out = torch.empty((nseg, 64), dtype=torch.int64, device="cuda")
    bad = []
    for g in (16, 32):
        fl = _lib.PP_SEG_OVERWRITE | (g << 8)
        us = _us_per_call(torch, lambda: _lib.check(lib.pp_count_segmented(
            buf.data_ptr(), offs.data_ptr(), nseg, 64, out.data_ptr(), fl, sp)))
        if us > 320:
            bad.append(f"G={g}: {us:.1f} us > 320")
    assert not bad, bad
