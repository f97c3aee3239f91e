"""The reference's own kernel-level test suite, restated for the B200 kernel.

Each test below carries the name of the reference test it restates
(pkg/tests/test_kernels.py, test_core.py, test_edges.py, test_acceptance.py,
file:line in the docstring) and checks the same property of the sm_100a
kernel, driven the way the reference drives a kernel: ``kernel.run(view, w,
counters)`` on a fresh counter list, or the ``pospopcnt`` entry point.  The
independent checks are the oracle's scalar restatement of core.py:82-96 and
its C port of NumbaKernel.run.  The reference's internal helpers
(count_tail, count_short, head_load) have no counterpart here; their
properties are checked through whole-array counts of the same lengths.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b200(cuda):
    torch, pp = cuda
    k = pp.get_kernel("b200")
    assert k.available()
    return pp, k


def fresh(k, view, w):
    return k.run(view, w, [0] * w)


def test_zeros_leave_counters(b200):
    """test_kernels.py:26-29."""
    pp, k = b200
    assert fresh(k, pp.InputView.of(bytes(16 * 1024)), 16) == [0] * 16


@pytest.mark.parametrize("n", (1, 1000, 1_000_000))
def test_repeating_word_pattern(b200, n):
    """test_kernels.py:32-37: bits 0 and 15 of every 16-bit word."""
    pp, k = b200
    assert fresh(k, pp.InputView.of(b"\x01\x80" * n), 16) == [n] + [0] * 14 + [n]


@pytest.mark.parametrize("w", (8, 16, 32, 64))
def test_oracle_spot_sweep(b200, oracle, rng, w):
    """test_kernels.py:40-50: lengths around the reference's block sizes at
    several offsets, against the scalar definition."""
    pp, k = b200
    step = w // 8
    data = rng.randbytes(3100)
    for n in (0, step, 5 * step, 119, 120, 121, 960, 1024, 2048, 2944):
        n -= n % step
        for off in (0, 1, 7, 9, 63):
            got = fresh(k, pp.InputView(data, off, n), w)
            assert got == oracle.scalar(data[off:off + n], w), (w, n, off)


def test_short_and_main_boundary(b200, oracle, rng):
    """test_kernels.py:53-62: straddle the 15-vector short-path threshold
    (r = 128 -> 16-byte vectors) and, for this kernel, its 16-byte body split
    and 32 KiB chunk."""
    pp, k = b200
    rb = k.r // 8
    data = rng.randbytes(2 * 32768 + 70)
    lengths = [15 * rb - 8, 15 * rb, 15 * rb + 8, 16 * rb - 8, 16 * rb, 16 * rb + 8,
               32768 - 8, 32768, 32768 + 8, 2 * 32768 - 8, 2 * 32768]
    for n in lengths:
        for off in (0, 3):
            got = fresh(k, pp.InputView(data, off, n), 64)
            assert got == oracle.scalar(data[off:off + n], 64), (n, off)


def test_streaming_equals_batch(b200, oracle, rng):
    """test_kernels.py:65-72: two runs into one counter list == one run."""
    pp, k = b200
    data = rng.randbytes(4096)
    for split in (0, 2, 722, 2048, 4096):
        c = [0] * 16
        k.run(pp.InputView(data, 0, split), 16, c)
        k.run(pp.InputView(data, split, 4096 - split), 16, c)
        assert c == oracle.scalar(data, 16), split


def test_alignment_invariance(b200, oracle, rng):
    """test_kernels.py:75-80: the same payload at 13 different offsets."""
    pp, k = b200
    payload = rng.randbytes(2000)
    want = oracle.scalar(payload, 8)
    for off in range(0, 64, 5):
        base = bytes(off) + payload + bytes(7)
        assert fresh(k, pp.InputView(base, off, len(payload)), 8) == want, off


def test_adjacent_memory_has_no_effect(b200, oracle, rng):
    """test_kernels.py:83-91: padding bytes 00 / ff / a5 around the view."""
    pp, k = b200
    payload = rng.randbytes(1500)
    res = []
    for pad in (b"\x00", b"\xff", b"\xa5"):
        base = pad * 37 + payload + pad * 37
        res.append(fresh(k, pp.InputView(base, 37, len(payload)), 8))
    assert res[0] == res[1] == res[2] == oracle.scalar(payload, 8)


def test_kernel_rejects_instrumentation(b200):
    """test_kernels.py:145-150 (the compiled kernel cannot take fa/probe)."""
    pp, k = b200
    with pytest.raises(ValueError):
        k.run(pp.InputView.of(b"\x00" * 8), 8, [0] * 8, fa=lambda *a: None)


def test_pospopcnt_entry_point(b200, oracle, rng):
    """test_kernels.py:188-198: default dispatch, by name, by object,
    accumulation into a given list, word-incomplete input rejected."""
    pp, k = b200
    data = rng.randbytes(1000)
    want = oracle.scalar(data, 8)
    assert pp.pospopcnt(data, 8) == want
    assert pp.pospopcnt(data, 8, kernel="b200") == want
    assert pp.pospopcnt(data, 8, kernel=k) == want
    c = [1] * 8
    pp.pospopcnt(data, 8, counters=c)
    assert c == [v + 1 for v in want]
    with pytest.raises(pp.InputLengthError):
        pp.pospopcnt(b"\x00" * 7, 64)


def test_buffer_types(b200, oracle, rng):
    """test_kernels.py:210-215, plus the device-side types of this build."""
    pp, k = b200
    import torch
    raw = rng.randbytes(2000)
    want = oracle.scalar(raw, 8)
    arr = np.frombuffer(raw, np.uint8)
    for data in (raw, bytearray(raw), memoryview(raw), arr, torch.from_numpy(arr.copy()),
                 torch.from_numpy(arr.copy()).cuda()):
        assert fresh(k, pp.InputView.of(data), 8) == want, type(data)


def test_kernel_equivalence_sampled(b200, oracle, rng):
    """test_kernels.py:218-225: sizes across the reference's block and flush
    boundaries, at offset 9, against its fastest kernel's C port."""
    pp, k = b200
    for n in (0, 8, 512, 4096, 65536, 122872, 122880, 131072, 1 << 20):
        data = np.frombuffer(rng.randbytes(n + 17), np.uint8)
        got = fresh(k, pp.InputView(data, 9, n), 16)
        assert got == oracle.hs512(data, 9, n, 16), n


def test_short_counter_array_rejected(b200, rng):
    """test_kernels.py:228-230."""
    pp, k = b200
    with pytest.raises(ValueError):
        pp.pospopcnt(rng.randbytes(16), 16, counters=[0] * 8)


def test_concurrent_calls_with_distinct_counters(b200, oracle, rng):
    """test_kernels.py:233-253: threads sharing one kernel object."""
    import threading
    pp, k = b200
    data = rng.randbytes(64 * 1024)
    want = oracle.scalar(data, 16)
    results, errors = [], []

    def work():
        try:
            outs = [k.run(pp.InputView.of(data), 16, [0] * 16) for _ in range(3)]
            results.append(all(o == want for o in outs))
        except Exception as exc:  # pragma: no cover - diagnostic only
            errors.append(exc)

    ths = [threading.Thread(target=work) for _ in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors and all(results) and len(results) == 4


def test_all_ones_word_and_empty_input(b200):
    """test_core.py:14-20."""
    pp, k = b200
    assert fresh(k, pp.InputView.of(b"\xff\xff"), 16) == [1] * 16
    c = [3] * 8
    assert k.run(pp.InputView.of(b""), 8, c) == [3] * 8


@pytest.mark.parametrize("w", (8, 16, 32, 64))
def test_conservation(b200, rng, w):
    """test_core.py:52-56: the counters sum to the popcount of the input."""
    pp, k = b200
    data = rng.randbytes(64 * (w // 8) * 1001)
    got = fresh(k, pp.InputView.of(data), w)
    assert pp.total_popcount_of(got) == int.from_bytes(data, "little").bit_count()


def test_counter_bound_and_determinism(b200, rng):
    """test_core.py:46-49, 59-64."""
    pp, k = b200
    data = rng.randbytes(100_000)
    a = fresh(k, pp.InputView.of(data), 16)
    assert a == fresh(k, pp.InputView.of(data), 16)
    assert all(0 <= x <= 50_000 for x in a)


@pytest.mark.parametrize("w", (8, 16, 32))
def test_width_refinement(b200, rng, w):
    """test_core.py:66-72: counting at 2w and folding == counting at w."""
    pp, k = b200
    data = rng.randbytes(40 * (w // 4) * 1003)
    wide = fresh(k, pp.InputView.of(data), 2 * w)
    narrow = fresh(k, pp.InputView.of(data), w)
    assert [wide[j] + wide[j + w] for j in range(w)] == narrow


def test_additivity(b200, oracle, rng):
    """test_core.py:75-80."""
    pp, k = b200
    a, b = rng.randbytes(30_001), rng.randbytes(71_003)
    c = fresh(k, pp.InputView.of(a), 8)
    k.run(pp.InputView.of(b), 8, c)
    assert c == oracle.scalar(a + b, 8)


@pytest.mark.parametrize("step", (1, 7, 64, 255, 1009))
def test_tail_lengths(b200, oracle, rng, step):
    """test_edges.py:77-83 (count_tail every length) and 113-119
    (count_short sweep): every short length, as whole arrays at an odd
    offset, so the kernel's head/tail lanes take all of them."""
    pp, k = b200
    data = rng.randbytes(1023 + 5)
    for n in range(0, 1024, step):
        assert fresh(k, pp.InputView(data, 5, n), 8) == oracle.scalar(data[5:5 + n], 8), n


def test_short_known_answers(b200):
    """test_edges.py:63-68, 71-74, 94-103."""
    pp, k = b200
    assert fresh(k, pp.InputView.of(bytes([0b10000001])), 8) == [1, 0, 0, 0, 0, 0, 0, 1]
    assert fresh(k, pp.InputView.of(b"\xff" * 8), 64) == [1] * 64
    assert fresh(k, pp.InputView.of(b"\x01\x00"), 16) == [1] + [0] * 15
    assert fresh(k, pp.InputView.of(bytes([0xFF, 0x00, 0x81])), 8) == [2, 1, 1, 1, 1, 1, 1, 2]


def test_criterion_4_overflow_discipline(b200):
    """test_acceptance.py:151-182: 256 MiB of 0xFF at w=16 (every counter
    134,217,728), counted on the device, far past any 16-bit discipline."""
    pp, k = b200
    import torch
    buf = torch.full((256 << 20,), 0xFF, dtype=torch.uint8, device="cuda")
    assert fresh(k, pp.InputView.of(buf), 16) == [134_217_728] * 16
