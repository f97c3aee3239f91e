"""GPU parity of the segmented (many-small-arrays) mode vs the CPU oracle.

Row s must equal the reference's count of segment s alone
(NumbaKernel.run on InputView(base, off[s], len_s), kernels.py:242-270).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def golden_digest(name):
    import json
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", "golden.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f)["digests"].get(name)


def test_c1_exhaustive_sweep_via_segments(cuda, oracle):
    """acceptance c1 (pkg/tests/test_acceptance.py:41-64): lengths 0..4096 x
    alignments 0..63 x every width, each case one segment of one launch.
    Case (a, n) is placed at device address = a mod 64 between poison gaps."""
    torch, pp = cuda
    import random
    rng = random.Random(20240)
    src = np.frombuffer(rng.randbytes(64 + 4096), np.uint8)
    from paper_2412_16370_b200 import _lib
    lib = _lib.load()
    for w in (8, 16, 32, 64):
        step = w // 8
        slot = 64 + 4096 + 64
        lens = np.arange(0, 4097, step)
        cases = [(a, int(n)) for a in range(64) for n in lens]
        host = np.full(len(cases) * slot, 0xA5, dtype=np.uint8)
        offs = np.empty(3 * len(cases) + 1, dtype=np.int64)
        real_rows = np.arange(len(cases)) * 3 + 1
        exp_offs = []
        for i, (a, n) in enumerate(cases):
            s = i * slot
            host[s + a:s + a + n] = src[a:a + n]
            offs[3 * i] = s
            offs[3 * i + 1] = s + a
            offs[3 * i + 2] = s + a + n
            exp_offs.append((s + a, s + a + n))
        offs[-1] = len(cases) * slot
        buf = torch.from_numpy(host).cuda()
        doffs = torch.from_numpy(offs).cuda()
        got = None
        # (lanes hint, extra flags): every shape, the default (0 = G 32), and
        # the hybrid split (short arrays one lane each) with two shapes
        for lanes, path in ((32, 0), (16, 0), (8, 0), (1, 0), (0, 0), (8, _lib.PP_SEG_HYBRID),
                            (32, _lib.PP_SEG_HYBRID)):
            # every launch shape must agree
            out = torch.zeros((3 * len(cases), w), dtype=torch.int64, device="cuda")
            rc = lib.pp_count_segmented(buf.data_ptr(), doffs.data_ptr(), 3 * len(cases), w,
                                        out.data_ptr(),
                                        _lib.PP_SEG_OVERWRITE | (lanes << 8) | path, None)
            _lib.check(rc)
            rows = out.cpu().numpy().view(np.uint64)[real_rows]
            if got is not None:
                assert np.array_equal(rows, got), (w, lanes)
            got = rows
        # oracle: the same views of the same bytes
        st = np.array([a for a, _ in exp_offs], dtype=np.uint64)
        en = np.array([b for _, b in exp_offs], dtype=np.uint64)
        want = oracle.views(host, st, en, w)
        assert np.array_equal(got, want), w
        # and against the reference's own outputs (golden digest, make_golden.py)
        dig = golden_digest(f"c1_sweep_w{w}")
        if dig is not None:
            import hashlib
            assert hashlib.sha256(np.ascontiguousarray(got).tobytes()).hexdigest() == \
                dig["sha256_u64_rows"], w


@pytest.mark.parametrize("lanes", (None, 1, 2, 4, 8, 16, 32))
def test_ragged_random_segments_poison(cuda, oracle, rng, lanes):
    torch, pp = cuda
    for w in (8, 16, 32, 64):
        step = w // 8
        lens = [rng.choice((0, step, 3 * step, 100 * step, rng.randrange(0, 9000) // step * step,
                            rng.randrange(0, 300_000) // step * step)) for _ in range(3000)]
        offs = np.zeros(len(lens) + 1, dtype=np.int64)
        offs[1:] = np.cumsum(lens)
        base = 5  # misaligned start of the whole batch
        host = np.frombuffer(rng.randbytes(int(offs[-1]) + base + 11), np.uint8).copy()
        buf = torch.from_numpy(host).cuda()
        view = pp.InputView(buf, base, int(offs[-1]))
        out = pp.pospopcnt_segmented(view, offs, w, lanes=lanes)
        want = oracle.segments(host, (offs + base).astype(np.uint64), w)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want), w
        # the hybrid split over the same mixed lengths, with every lane hint:
        # G = 2 demotes to one lane per segment on CSR offsets, which must
        # drop the split (rows of long segments were never written)
        hy = pp.pospopcnt_segmented(view, offs, w, lanes=lanes, hybrid=True)
        assert np.array_equal(hy.cpu().numpy().view(np.uint64), want), w
        # accumulate semantics
        pp.pospopcnt_segmented(view, offs, w, out=out, lanes=lanes)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), 2 * want), w
        pp.pospopcnt_segmented(view, offs, w, out=out, accumulate=False, lanes=lanes)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want), w


def test_tiny_arrays_one_lane_each(cuda, oracle, rng):
    """Arrays of a few words (C4's short lengths, batched): the automatic
    shape is one lane per array (pp_seglane_kernel).  Fixed sizes at every
    byte offset of the batch, and ragged tiny arrays from host offsets."""
    torch, pp = cuda
    host = np.frombuffer(rng.randbytes((1 << 21) + 64), np.uint8).copy()
    buf = torch.from_numpy(host).cuda()
    for w in (8, 16, 32, 64):
        step = w // 8
        for seg in sorted({step, 8, 24, 136, 256}):
            if seg % step:
                continue
            for off in (0, 1, 3, 7):
                nseg = 4099 if seg > 64 else 20011
                view = pp.InputView(buf, off, nseg * seg)
                out = pp.pospopcnt_fixed(view, seg, w)
                offs = (np.arange(nseg + 1, dtype=np.uint64) * seg + off)
                want = oracle.segments(host, offs, w)
                assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (w, seg, off)
        lens = [rng.randrange(0, 257) // step * step for _ in range(7777)]
        offs = np.zeros(len(lens) + 1, dtype=np.int64)
        offs[1:] = np.cumsum(lens)
        view = pp.InputView(buf, 3, int(offs[-1]))
        out = pp.pospopcnt_segmented(view, offs, w)
        want = oracle.segments(host, (offs + 3).astype(np.uint64), w)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want), w
        # device-side offsets: the shape is chosen during validation
        out = pp.pospopcnt_segmented(view, torch.from_numpy(offs).cuda(), w)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want), w


@pytest.mark.parametrize("lanes", (1, 8, 32))
def test_config_c4_segmented_batch(cuda, oracle, lanes):
    """262,144 independent 4 KiB arrays of Bernoulli(0.01) bits, w=64."""
    torch, pp = cuda
    from paper_2412_16370_b200 import gen
    nseg, seg = 262_144, 4096
    buf = gen.generate("bernoulli", nseg * seg, 0xC4 + 1, q=655)
    out = pp.pospopcnt_fixed(buf, seg, 64, lanes=lanes)
    got = out.cpu().numpy().view(np.uint64)
    host = buf.cpu().numpy()
    offs = np.arange(nseg + 1, dtype=np.uint64) * seg
    want = oracle.segments(host, offs, 64)
    assert np.array_equal(got, want)
    # the fixed and CSR entry points agree
    out2 = pp.pospopcnt_segmented(buf, offs.astype(np.int64), 64, lanes=lanes)
    assert np.array_equal(out2.cpu().numpy().view(np.uint64), want)


def test_segment_errors(cuda):
    torch, pp = cuda
    buf = torch.zeros(100, dtype=torch.uint8, device="cuda")
    with pytest.raises(pp.InputLengthError):
        pp.pospopcnt_segmented(buf, [0, 3, 8], 16)
    with pytest.raises(ValueError):
        pp.pospopcnt_segmented(buf, [0, 8, 4], 8)
    with pytest.raises(ValueError):
        pp.pospopcnt_segmented(buf, [0, 200], 8)
    with pytest.raises(pp.InputLengthError):
        pp.pospopcnt_fixed(buf, 3, 16)
    assert pp.pospopcnt_segmented(buf, [0], 8).shape == (0, 8)


@pytest.mark.parametrize("lanes", (None, 1, 8, 32))
def test_batch_of_separate_arrays(cuda, oracle, rng, lanes):
    """pospopcnt_batch: arrays in separate allocations (and views at odd
    offsets inside them), each row == that array's own count; every array is
    read only within its own bounds (exact-size allocations)."""
    torch, pp = cuda
    for w in (8, 16, 64):
        step = w // 8
        arrays, hosts = [], []
        for i in range(600):
            n = rng.choice((0, step, 3 * step, 17 * step, 200 * step,
                            rng.randrange(0, 20000) // step * step))
            off = rng.randrange(0, 16)
            host = np.frombuffer(rng.randbytes(off + n), np.uint8)
            t = torch.from_numpy(host.copy()).cuda()  # exactly off + n bytes
            arrays.append(pp.InputView(t, off, n) if off else t)
            hosts.append(host[off:])
        out = pp.pospopcnt_batch(arrays, w, lanes=lanes)
        got = out.cpu().numpy().view(np.uint64)
        for i, h in enumerate(hosts):
            assert list(got[i]) == oracle.scalar(h.tobytes(), w), (w, i)
        # accumulate into the same rows
        pp.pospopcnt_batch(arrays, w, out=out, lanes=lanes)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), 2 * got)
    with pytest.raises(pp.InputLengthError):
        pp.pospopcnt_batch([torch.zeros(3, dtype=torch.uint8, device="cuda")], 16)


def test_ticket_batches_many_segments(cuda, oracle):
    """Launches with more than 49,152 groups batch T > 1 groups per scheduler
    ticket (seg_batch_groups); explicit PP_SEG_BATCH hints 1 / 5 / 63 too.
    Every shape must stay exact, including a last batch that is partial."""
    torch, pp = cuda
    from paper_2412_16370_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(31)
    nseg = 300_007
    lens = rng.integers(0, 2048 // 8, nseg) * 8
    offs = np.zeros(nseg + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens)
    host = rng.integers(0, 256, int(offs[-1]) + 16, dtype=np.uint8)
    buf = torch.from_numpy(host).cuda()
    d = torch.from_numpy(offs).cuda()
    want = oracle.segments(host, offs.astype(np.uint64), 64)
    out = torch.empty((nseg, 64), dtype=torch.int64, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    for lanes in (8, 16, 32):
        for t in (0, 1, 5, 63):
            out.fill_(-1)
            fl = _lib.PP_SEG_OVERWRITE | (lanes << 8) | (t << _lib.PP_SEG_BATCH_SHIFT)
            _lib.check(lib.pp_count_segmented(buf.data_ptr(), d.data_ptr(), nseg, 64,
                                              out.data_ptr(), fl, sp))
            assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (lanes, t)


@pytest.mark.parametrize("lanes", (None, 8, 16, 32))
def test_segment_plan_exact(cuda, oracle, lanes):
    """SegmentPlan (length-sorted processing order, pp_count_segmented_order)
    must give the same rows as the plain segmented count: ragged lengths
    incl. empty, tiny (hybrid pass) and long segments, misaligned base,
    overwrite and accumulate, every width."""
    torch, pp = cuda
    rng = np.random.default_rng(77)
    for w in (8, 16, 32, 64):
        step = w // 8
        lens = np.concatenate([rng.integers(0, 8192 // step, 20_000) * step,
                               np.zeros(7, np.int64), np.full(50, 3 * step),
                               rng.integers(0, 300_000 // step, 40) * step])
        rng.shuffle(lens)
        offs = np.zeros(lens.size + 1, dtype=np.int64)
        offs[1:] = np.cumsum(lens)
        base = 3
        host = rng.integers(0, 256, int(offs[-1]) + base + 5, dtype=np.uint8)
        buf = torch.from_numpy(host).cuda()
        view = pp.InputView(buf, base, int(offs[-1]))
        want = oracle.segments(host, (offs + base).astype(np.uint64), w)
        plan = pp.SegmentPlan(offs, device="cuda", lanes=lanes)
        out = pp.pospopcnt_segmented(view, None, w, plan=plan)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (w, plan.lanes)
        plan.count(view, w, out=out)  # accumulate
        assert np.array_equal(out.cpu().numpy().view(np.uint64), 2 * want), w
        tiny = pp.SegmentPlan(np.where(rng.random(5000) < 0.9, 64, 4096).cumsum(), device="cuda")
        assert tiny.hybrid and tiny.lanes == 32
    with pytest.raises(ValueError):
        pp.SegmentPlan([0, 8, 4])


def test_plan_auto_cache(cuda, oracle):
    """A ragged segmentation counted again with the same offsets gets a
    cached SegmentPlan (second sighting), rows unchanged; an in-place write
    to a device offsets tensor, or different host offsets, never reuse a
    stale plan; plan=False opts out."""
    torch, pp = cuda
    from paper_2412_16370_b200 import segmented as S
    S._PLANS.clear()
    rng = np.random.default_rng(5)
    w = 32
    lens = rng.integers(0, 6000 // 4, 4000) * 4
    offs = np.zeros(lens.size + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens)
    host = rng.integers(0, 256, int(offs[-1]) + 16, dtype=np.uint8)
    buf = torch.from_numpy(host).cuda()
    want = oracle.segments(host, offs.astype(np.uint64), w)
    for src in ("host", "device"):
        S._PLANS.clear()
        o = offs.copy() if src == "host" else torch.as_tensor(offs, device="cuda")
        for i in range(4):
            out = pp.pospopcnt_segmented(buf, o, w)
            assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (src, i)
        built, hits = S._PLANS.stats
        assert built == 1 and hits == 2, (src, S._PLANS.stats)
        # a different segmentation
        o2 = offs.copy()
        o2[1] = 0  # segment 0 empty, segment 1 longer
        want2 = oracle.segments(host, o2.astype(np.uint64), w)
        if src == "device":
            o.copy_(torch.as_tensor(o2))  # in place: version bump
            o2 = o
        out = pp.pospopcnt_segmented(buf, o2, w)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want2), src
        assert S._PLANS.stats[1] == 2  # no stale hit
    out = pp.pospopcnt_segmented(buf, offs, w, plan=False)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want)
