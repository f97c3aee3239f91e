"""GPU parity: the sm_100a path (through the C ABI) vs the CPU oracle.

Bit-exact integer counts are the bar.  Cases mirror the reference's own
kernel and acceptance tests (pkg/tests/test_kernels.py, test_acceptance.py):
known answers, length x offset sweeps, alignment / adjacent-memory
invariance, streaming = batch, conservation, the all-ones overflow check
(scaled past 2^32 words), and the BASELINE configs at full size.
"""

import ctypes
import threading

import numpy as np
import pytest

from conftest import oracle_bits

pytestmark = pytest.mark.gpu

MIB = 1 << 20


def dev_bytes(torch, data, offset=0, pad=0, fill=0):
    """Place host bytes at `offset` inside a padded CUDA buffer; returns (buf, view)."""
    import paper_2412_16370_b200 as pp
    raw = np.frombuffer(bytes(data), dtype=np.uint8)
    host = np.full(offset + raw.size + pad, fill, dtype=np.uint8)
    host[offset:offset + raw.size] = raw
    buf = torch.from_numpy(host).cuda()
    return buf, pp.InputView(buf, offset, raw.size)


def count(torch, pp, view, w):
    c = torch.zeros(w, dtype=torch.int64, device="cuda")
    pp.pospopcnt(view, w, counters=c)
    return [int(x) for x in c.cpu().numpy().view(np.uint64)]


# ----------------------------------------------------------- known answers
def test_known_answers(cuda):
    torch, pp = cuda
    assert pp.pospopcnt(torch.tensor([1, 128], dtype=torch.uint8).cuda(), 16) == \
        [1] + [0] * 14 + [1]
    assert pp.pospopcnt(torch.tensor([255, 255], dtype=torch.uint8).cuda(), 16) == [1] * 16
    assert pp.pospopcnt(torch.tensor([0xFF, 0x00, 0x81], dtype=torch.uint8).cuda(), 8) == \
        [2, 1, 1, 1, 1, 1, 1, 2]
    assert pp.pospopcnt(torch.tensor([0x0F], dtype=torch.uint8).cuda(), 8) == \
        [1, 1, 1, 1, 0, 0, 0, 0]
    for n in (1, 1000, 1_000_000):
        buf, view = dev_bytes(torch, b"\x01\x80" * n)
        assert count(torch, pp, view, 16) == [n] + [0] * 14 + [n], n
    z = torch.zeros(16 * 1024, dtype=torch.uint8, device="cuda")
    for w in (8, 16, 32, 64):
        assert pp.pospopcnt(z, w) == [0] * w
        assert pp.pospopcnt(z[:0], w) == [0] * w


def test_host_bytes_entry(cuda, rng):
    """bytes / bytearray / memoryview / numpy go through the pipelined host path."""
    torch, pp = cuda
    raw = rng.randbytes(100_000)
    want = oracle_bits(raw, 8)
    for data in (raw, bytearray(raw), memoryview(raw), np.frombuffer(raw, np.uint8)):
        assert pp.pospopcnt(data, 8) == want
    c = [1] * 8
    pp.pospopcnt(raw, 8, counters=c)
    assert c == [v + 1 for v in want]
    big = np.frombuffer(rng.randbytes(70 * MIB + 24), np.uint8)  # > 2 staging chunks
    from oracle import oracle as O
    assert pp.pospopcnt(pp.InputView(big, 3, 70 * MIB + 16), 16) == \
        O.hs512(big, 3, 70 * MIB + 16, 16, threads=8)


# ------------------------------------------------- sweeps vs the oracle
@pytest.mark.parametrize("w", (8, 16, 32, 64))
def test_spot_sweep_lengths_offsets(cuda, oracle, rng, w):
    """test_kernels.py:40-50 sizes plus chunk-boundary sizes of the B200 kernel."""
    torch, pp = cuda
    step = w // 8
    data = rng.randbytes(3 * (1 << 16) + 200)
    host = np.frombuffer(data, np.uint8)
    buf = torch.from_numpy(host.copy()).cuda()
    sizes = [0, step, 5 * step, 119, 120, 121, 960, 1024, 2048, 2944, 4096, 32768 - 8,
             32768, 32768 + 8, 65536, 65536 + 24, 3 * (1 << 16)]
    for n in sizes:
        n -= n % step
        for off in (0, 1, 3, 7, 9, 15, 16, 63):
            if off + n > len(data):
                continue
            want = oracle.hs512(host, off, n, w)
            got = count(torch, pp, pp.InputView(buf, off, n), w)
            assert got == want, (w, n, off)


def test_alignment_invariance_and_poison(cuda, rng):
    """test_kernels.py:75-91: offset and adjacent bytes never change the result."""
    torch, pp = cuda
    payload = rng.randbytes(70_000)
    want = oracle_bits(payload, 8)
    for off in range(0, 64, 5):
        for fill in (0x00, 0xFF, 0xA5):
            buf, view = dev_bytes(torch, payload, off, pad=37, fill=fill)
            assert count(torch, pp, view, 8) == want, (off, fill)


def test_streaming_equals_batch(cuda, oracle, rng):
    """test_kernels.py:65-72 / acceptance c5: split counts add up exactly."""
    torch, pp = cuda
    data = rng.randbytes(1 << 20)
    buf = torch.from_numpy(np.frombuffer(data, np.uint8).copy()).cuda()
    want = oracle.hs512(data, 0, len(data), 16)
    for split in (0, 2, 722, 2048, 32768 + 6, 1 << 19, 1 << 20):
        c = torch.zeros(16, dtype=torch.int64, device="cuda")
        pp.pospopcnt(pp.InputView(buf, 0, split), 16, counters=c)
        pp.pospopcnt(pp.InputView(buf, split, len(data) - split), 16, counters=c)
        assert [int(x) for x in c.cpu()] == want, split


def test_conservation_random_cases(cuda, rng):
    """acceptance c5 conservation: sum of counters = popcount of the input."""
    torch, pp = cuda
    for case in range(200):
        w = (8, 16, 32, 64)[case % 4]
        n = rng.randrange(0, 200_000 // (w // 8) + 1) * (w // 8)
        data = rng.randbytes(n)
        off = rng.randrange(0, 16)
        buf, view = dev_bytes(torch, data, off, pad=rng.randrange(0, 9), fill=0xFF)
        got = count(torch, pp, view, w)
        assert sum(got) == int.from_bytes(data, "little").bit_count(), (w, n, off)


# --------------------------------------------------------- exactness at scale
def test_all_ones_past_2_32_words(cuda):
    """acceptance c4 (256 MiB all-ones at w=16) scaled to 5 GiB at w=8:
    every counter is 5*2^30 > 2^32, so any 32-bit truncation shows."""
    torch, pp = cuda
    buf = torch.full((256 * MIB,), 0xFF, dtype=torch.uint8, device="cuda")
    c = torch.zeros(16, dtype=torch.int64, device="cuda")
    pp.pospopcnt(buf, 16, counters=c)
    assert [int(x) for x in c.cpu()] == [134_217_728] * 16
    del buf
    n = 5 << 30
    big = torch.full((n,), 0xFF, dtype=torch.uint8, device="cuda")
    c = torch.zeros(8, dtype=torch.int64, device="cuda")
    pp.pospopcnt(big, 8, counters=c)
    assert [int(x) for x in c.cpu()] == [n] * 8
    del big
    torch.cuda.empty_cache()


def test_generators_match_cpu_twins(cuda, oracle):
    torch, pp = cuda
    from paper_2412_16370_b200 import gen
    n = 1 << 16
    for off in (0, 12345):
        assert np.array_equal(gen.generate("uniform", n, 7, word_offset=off).cpu().numpy(),
                              oracle.gen_uniform(n, 7, off))
        assert np.array_equal(gen.generate("bernoulli", n, 8, word_offset=off, q=655).cpu().numpy(),
                              oracle.gen_bernoulli(n, 8, 655, off))
        assert np.array_equal(gen.generate("blocks", n, 9, word_offset=off,
                                           block_bytes=4096).cpu().numpy(),
                              oracle.gen_blocks(n, 9, 4096, off))
        assert np.array_equal(gen.generate("onehot32", n, 10, word_offset=off).cpu().numpy(),
                              oracle.gen_onehot32(n, 10, word_offset=off))
    ones = gen.generate("bernoulli", 4096, 1, q=65536).cpu().numpy()
    assert (ones == 0xFF).all()


def _full_size(torch, pp, oracle, kind, nbytes, w, seed, **kw):
    from paper_2412_16370_b200 import gen
    buf = gen.generate(kind, nbytes, seed, **kw)
    c = torch.zeros(w, dtype=torch.int64, device="cuda")
    pp.pospopcnt(buf, w, counters=c)
    got = [int(x) for x in c.cpu()]
    host = buf.cpu().numpy()
    del buf
    return got, host


def test_config_c1_w16_2mib(cuda, oracle):
    torch, pp = cuda
    got, host = _full_size(torch, pp, oracle, "uniform", 2 * MIB, 16, 0xC1)
    assert got == oracle.hs512(host, 0, host.size, 16)
    assert got == oracle.scalar(host, 16)


def test_config_c2_w8_1gib(cuda, oracle):
    torch, pp = cuda
    got, host = _full_size(torch, pp, oracle, "uniform", 1 << 30, 8, 0xC2)
    assert got == oracle.hs512(host, 0, host.size, 8, threads=16)


def test_config_c3_w32_onehot_4gib(cuda, oracle):
    torch, pp = cuda
    nbytes = 4 << 30
    got, host = _full_size(torch, pp, oracle, "onehot32", nbytes, 32, 0xC3)
    assert sum(got) == nbytes // 4  # exactly one bit per word
    assert got == oracle.hs512(host, 0, host.size, 32, threads=16)
    assert got[0] > got[1] > got[8] > got[31] > 0  # Zipf-shaped


def test_config_c4_w64_short_unaligned(cuda, oracle):
    torch, pp = cuda
    from paper_2412_16370_b200 import gen
    lengths = (1, 3, 17, 255, 512, 8192, 131072, 8388608)
    buf = gen.generate("bernoulli", 64 * MIB + 64, 0xC4, q=655)
    host = buf.cpu().numpy()
    for n in lengths:
        for off in range(1, 8):
            nb = 8 * n
            got = count(torch, pp, pp.InputView(buf, off, nb), 64)
            assert got == oracle.hs512(host, off, nb, 64, threads=8), (n, off)


def test_config_c5_shard_w16(cuda, oracle):
    """One 1 GiB shard of the 64 GiB C5 array (word_offset places it mid-array)."""
    torch, pp = cuda
    got, host = _full_size(torch, pp, oracle, "blocks", 1 << 30, 16, 0xC5,
                           word_offset=(3 << 30) // 8)
    assert got == oracle.hs512(host, 0, host.size, 16, threads=16)


# ----------------------------------------------------------- API behaviour
def test_device_counters_accumulate_and_errors(cuda, rng):
    torch, pp = cuda
    data = rng.randbytes(4096)
    buf, view = dev_bytes(torch, data)
    c = torch.ones(8, dtype=torch.int64, device="cuda")
    pp.pospopcnt(view, 8, counters=c)
    pp.pospopcnt(view, 8, counters=c)
    want = oracle_bits(data, 8)
    assert [int(x) for x in c.cpu()] == [1 + 2 * v for v in want]
    with pytest.raises(pp.InputLengthError):
        pp.pospopcnt(buf[:7], 64)
    with pytest.raises(ValueError):
        pp.pospopcnt(buf, 12)
    with pytest.raises(ValueError):
        pp.pospopcnt(buf, 16, counters=[0] * 8)
    longer = [0] * 20
    pp.pospopcnt(view, 16, counters=longer)
    assert longer[16:] == [0] * 4


def test_c_abi_rejects_host_pointers(cuda):
    torch, pp = cuda
    from paper_2412_16370_b200 import _lib
    lib = _lib.load()
    host = np.zeros(64, dtype=np.uint8)
    dc = torch.zeros(8, dtype=torch.int64, device="cuda")
    rc = lib.pp_count(host.ctypes.data, 64, 8, dc.data_ptr(), None)
    assert rc == _lib.PP_EARG
    assert b"device" in lib.pp_last_error() or b"CUDA" in lib.pp_last_error()
    rc = lib.pp_count(dc.data_ptr(), 64, 12, dc.data_ptr(), None)
    assert rc == _lib.PP_EWIDTH
    # and the host entry point rejects device memory (it would memcpy from it)
    out = np.zeros(64, dtype=np.uint64)
    dd = torch.zeros(64, dtype=torch.uint8, device="cuda")
    assert lib.pp_count_host(dd.data_ptr(), 64, 8, out.ctypes.data) == _lib.PP_EARG
    assert lib.pp_count_host(host.ctypes.data, 64, 8, dc.data_ptr()) == _lib.PP_EARG


def test_concurrent_threads_distinct_counters(cuda, rng):
    """test_kernels.py:233-253."""
    torch, pp = cuda
    data = rng.randbytes(1 << 20)
    want = oracle_bits(data[:4096], 16)
    full_want = None
    from oracle import oracle as O
    full_want = O.hs512(data, 0, len(data), 16)
    buf, view = dev_bytes(torch, data)
    results, errors = [], []

    def work(use_host):
        try:
            outs = []
            for _ in range(5):
                if use_host:
                    outs.append(pp.pospopcnt(data, 16))
                else:
                    outs.append(pp.pospopcnt(view, 16))
            results.append(all(o == full_want for o in outs))
        except Exception as exc:  # pragma: no cover
            errors.append(exc)

    ths = [threading.Thread(target=work, args=(i % 2 == 0,)) for i in range(6)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors and all(results) and len(results) == 6
    assert want == oracle_bits(data[:4096], 16)


def test_all_widths_from_one_frame_pass(cuda, oracle, rng):
    """one pass, every width, any alignment (incl. words
    straddling 16-byte vectors)."""
    torch, pp = cuda
    host = np.frombuffer(rng.randbytes((1 << 20) + 64), np.uint8)
    buf = torch.from_numpy(host.copy()).cuda()
    for off, n in ((0, 1 << 20), (3, (1 << 20) - 8), (5, 1000), (7, 6), (1, 3), (0, 0)):
        got = pp.pospopcnt_all_widths(pp.InputView(buf, off, n))
        for w, cnt in got.items():
            assert cnt == oracle.hs512(host, off, n, w), (off, n, w)
        assert set(got) == {w for w in (8, 16, 32, 64) if n % (w // 8) == 0}
    assert pp.pospopcnt_all_widths(host[3:3 + 4096].tobytes(), widths=(16,)) == \
        {16: oracle.hs512(host, 3, 4096, 16)}


def test_cuda_graph_capture_and_replay(cuda, oracle, rng):
    """pp_count is capture-safe: a captured count replays on new data."""
    torch, pp = cuda
    host = np.frombuffer(rng.randbytes(3 << 20), np.uint8)
    buf = torch.from_numpy(host.copy()).cuda()
    cnt = torch.zeros(16, dtype=torch.int64, device="cuda")
    pp.pospopcnt(buf, 16, counters=cnt)  # warm (device info, attributes)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pp.pospopcnt(pp.InputView(buf, 5, 2 << 20), 16, counters=cnt)
    cnt.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    want = oracle.hs512(host, 5, 2 << 20, 16)
    assert [int(x) for x in cnt.cpu()] == [2 * v for v in want]
    host2 = np.frombuffer(rng.randbytes(3 << 20), np.uint8)
    buf.copy_(torch.from_numpy(host2.copy()))
    cnt.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert [int(x) for x in cnt.cpu()] == oracle.hs512(host2, 5, 2 << 20, 16)


def test_pdl_contract_generate_then_count(cuda, oracle):
    """The device generators trigger dependents at entry, so each pp_count
    (PDL-launched below 512 MiB) may start while its input is still being
    written; griddepcontrol.wait before the first read must make every
    count see the complete input."""
    torch, pp = cuda
    from paper_2412_16370_b200 import gen
    n = 64 << 20
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    cnt = torch.zeros((12, 16), dtype=torch.int64, device="cuda")
    for i in range(12):  # no host sync in between
        gen.generate("uniform", n, 1000 + i, out=buf)
        pp.pospopcnt(buf, 16, counters=cnt[i])
    codes = torch.empty(n, dtype=torch.uint8, device="cuda")
    ccnt = torch.zeros((4, 32), dtype=torch.int64, device="cuda")
    for i in range(4):
        gen.generate("codes8", n, 2000 + i, out=codes)
        pp.pospopcnt_categories(codes, 32, counters=ccnt[i])
    torch.cuda.synchronize()
    for i in range(12):
        host = oracle.gen_uniform(n, 1000 + i)
        assert [int(x) for x in cnt[i].cpu()] == oracle.hs512(host, 0, n, 16, threads=8), i
    for i in range(4):
        assert [int(x) for x in ccnt[i].cpu()] == oracle.categories(oracle.gen_codes8(n, 2000 + i), 32)


def test_input_ready_back_to_back(cuda, oracle):
    """pp_count_ex(PP_COUNT_INPUT_READY): counts of inputs written before the
    previous kernel on the stream may start loading during that kernel's
    tail.  Back to back over distinct resident inputs (static and ticketed
    chunk orders, unaligned views, alternating with plain counts into the
    same counters): every count exact, counters accumulate.  Unknown flags
    are an argument error."""
    torch, pp = cuda
    from paper_2412_16370_b200 import _lib, gen
    from paper_2412_16370_b200.kernels import count_device
    lib = _lib.load()
    sizes = (2 << 20, 64 << 20, 256 << 20)  # static order / static / tickets
    bufs = [gen.generate("uniform", n + 64, 3000 + i) for i, n in enumerate(sizes)]
    torch.cuda.synchronize()
    cnt = torch.zeros((len(sizes), 64), dtype=torch.int64, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    reps = 6
    for r in range(reps):
        for i, (n, b) in enumerate(zip(sizes, bufs)):
            off = (r * 5 + i) % 7
            if r % 2:
                count_device(b.data_ptr() + off, n, 64, cnt[i].data_ptr(), sp, input_ready=True)
            else:
                pp.pospopcnt(pp.InputView(b, off, n), 64, counters=cnt[i], input_ready=True)
            _lib.check(lib.pp_count(b.data_ptr(), n, 64, cnt[i].data_ptr(), sp))
    torch.cuda.synchronize()
    for i, (n, b) in enumerate(zip(sizes, bufs)):
        host = b.cpu().numpy()
        want = [0] * 64
        for r in range(reps):
            off = (r * 5 + i) % 7
            for j, v in enumerate(oracle.hs512(host, off, n, 64, threads=8)):
                want[j] += v
        for j, v in enumerate(oracle.hs512(host, 0, n, 64, threads=8)):
            want[j] += reps * v
        assert [int(x) for x in cnt[i].cpu()] == want, n
    with pytest.raises(ValueError):
        _lib.check(lib.pp_count_ex(bufs[0].data_ptr(), 64, 8, cnt[0].data_ptr(), 2, sp))


def test_dynamic_schedule_boundaries_and_streams(cuda, oracle):
    """The ticketed chunk order (inputs >= 4096 chunks of 32 KiB = 128 MiB):
    lengths either side of the switch, odd offsets and tails, concurrent
    launches on several streams (one scheduler slot per stream), a CUDA
    graph capture of a large count (static order inside captures), and the
    fixed-segment TMA kernel sharing a stream's slot with the count kernel."""
    torch, pp = cuda
    from paper_2412_16370_b200 import gen
    n = (160 << 20) + 64
    buf = gen.generate("uniform", n, 0xD1)
    host = buf.cpu().numpy()
    mib128 = 128 << 20
    cases = [(0, mib128 - 32768), (0, mib128), (3, mib128 + 40), (16, mib128 + 32768 + 8),
             (7, (160 << 20) - 8)]
    for off, ln in cases:
        want = oracle.hs512(host, off, ln, 8)
        c = torch.zeros(8, dtype=torch.int64, device="cuda")
        for _ in range(3):  # back to back on one stream: the slot re-arms each time
            pp.pospopcnt(pp.InputView(buf, off, ln), 8, counters=c)
        assert [int(x) for x in c.cpu()] == [3 * v for v in want], (off, ln)
    # several streams at once, each with its own slot
    streams = [torch.cuda.Stream() for _ in range(4)]
    outs = [torch.zeros(16, dtype=torch.int64, device="cuda") for _ in streams]
    torch.cuda.synchronize()
    for rep in range(3):
        for i, (st, o) in enumerate(zip(streams, outs)):
            with torch.cuda.stream(st):
                pp.pospopcnt(pp.InputView(buf, 8 * i, mib128 + 4096 * i), 16, counters=o)
    torch.cuda.synchronize()
    for i, o in enumerate(outs):
        want = oracle.hs512(host, 8 * i, mib128 + 4096 * i, 16)
        assert [int(x) for x in o.cpu()] == [3 * v for v in want], i
    # two host threads launching onto ONE stream: each launch's ticket base is
    # handed out and the launch enqueued in one critical section
    import threading
    shared = torch.cuda.Stream()
    outs2 = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(2)]

    def hammer(i):
        with torch.cuda.stream(shared):
            for _ in range(6):
                pp.pospopcnt(pp.InputView(buf, 0, mib128 + 8 * i), 8, counters=outs2[i])

    ths = [threading.Thread(target=hammer, args=(i,)) for i in range(2)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    torch.cuda.synchronize()
    for i, o in enumerate(outs2):
        assert [int(x) for x in o.cpu()] == [6 * v for v in oracle.hs512(host, 0, mib128 + 8 * i, 8)]
    # graph capture of a large count: replays stay exact
    c = torch.zeros(32, dtype=torch.int64, device="cuda")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pp.pospopcnt(pp.InputView(buf, 0, 150 << 20), 32, counters=c)
    c.zero_()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    assert [int(x) for x in c.cpu()] == [2 * v for v in oracle.hs512(host, 0, 150 << 20, 32)]
    # the segmented TMA kernel and the count kernel alternating on one stream
    rows = None
    for _ in range(2):
        rows = pp.pospopcnt_fixed(buf[: 160 << 20], 4096, 64)
        c64 = torch.zeros(64, dtype=torch.int64, device="cuda")
        pp.pospopcnt(buf[: 160 << 20], 64, counters=c64)
    got_rows = rows.cpu().numpy().view(np.uint64)
    assert np.array_equal(got_rows.sum(axis=0), np.array(oracle.hs512(host, 0, 160 << 20, 64),
                                                         dtype=np.uint64))
    assert [int(x) for x in c64.cpu()] == oracle.hs512(host, 0, 160 << 20, 64)


def _raw_streams(n):
    """n fresh CUDA streams (cudaStreamCreateWithFlags through cuda-python):
    torch.cuda.Stream() recycles a pool of 32 per device, which never gets
    past the scheduler's 256 slots."""
    import torch
    from cuda.bindings import runtime as rt
    out = []
    for _ in range(n):
        err, h = rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking)
        assert err == rt.cudaError_t.cudaSuccess, err
        out.append((int(h), torch.cuda.ExternalStream(int(h))))
    return out


def _sched_stats():
    import ctypes
    from paper_2412_16370_b200 import _lib
    out = (ctypes.c_uint64 * 4)()
    assert _lib.load().pp_sched_stats(out) == 0
    return list(out)  # handed out, taken over, all-busy static, dynamic launches


def test_scheduler_slots_reused_by_new_streams(cuda, oracle):
    """More streams than scheduler slots (256 per device): a new stream takes
    over a slot whose last launch has completed; with every slot busy it
    falls back to the static order.  Real streams (not torch's pool of 32),
    and pp_sched_stats proves both paths ran.  Every count must stay exact,
    including on the old streams afterwards."""
    torch, pp = cuda
    from cuda.bindings import runtime as rt
    from paper_2412_16370_b200 import gen
    n = 160 << 20  # > 128 MiB: the dynamically scheduled path
    buf = gen.generate("uniform", n, 0x5107)
    want = oracle.hs512(buf.cpu().numpy(), 0, n, 8)
    s0 = _sched_stats()
    streams = _raw_streams(300)
    keep = []
    # every counter tensor is zeroed on the stream that counts into it: 600
    # streams share a few hardware queues, so a zero-fill on another stream
    # can sit behind a gated launch and land after the count
    for i, (h, s) in enumerate(streams):  # sequential: each launch done before the next
        with torch.cuda.stream(s):
            c = torch.zeros(8, dtype=torch.int64, device="cuda")
            pp.pospopcnt(buf, 8, counters=c)
        s.synchronize()
        assert [int(x) for x in c.cpu()] == want, i
        if i % 50 == 0:
            keep.append(s)
    s1 = _sched_stats()
    # the first 256 - (slots used before) streams got fresh slots, the rest
    # took over completed ones
    assert s1[1] - s0[1] >= 300 - 256, (s0, s1)
    busy = _raw_streams(300)
    # every stream waits on one host-released gate: all their launches are
    # in flight at once, so every slot is busy and the later ones must take
    # the static order.  The gate is a stream wait on a pinned host word
    # (cuStreamWaitValue32) that this thread sets once the launches are
    # queued -- no race against a timed blocker kernel.
    from cuda.bindings import driver as drv
    word = torch.zeros(1, dtype=torch.int32).pin_memory()
    gate = torch.cuda.Event()
    blocker = torch.cuda.Stream()
    err, = drv.cuStreamWaitValue32(blocker.cuda_stream, word.data_ptr(), 1,
                                   drv.CUstreamWaitValue_flags.CU_STREAM_WAIT_VALUE_EQ)
    assert err == drv.CUresult.CUDA_SUCCESS, err
    outs = []
    import threading

    def release():
        word[0] = 1
    watchdog = threading.Timer(30.0, release)  # a blocked host call must not hang the GPU
    watchdog.daemon = True
    watchdog.start()
    try:
        gate.record(blocker)
        for h, s in busy:
            s.wait_event(gate)
            with torch.cuda.stream(s):
                c = torch.zeros(8, dtype=torch.int64, device="cuda")
                pp.pospopcnt(buf, 8, counters=c)
            outs.append((s, c))
        s2 = _sched_stats()
        assert not gate.query()  # still closed: every queued launch is pending
    finally:
        release()  # open the gate whatever happened above
        watchdog.cancel()
    assert s2[2] > s1[2], (s1, s2)  # all-busy launches used the static order
    for s in keep:  # streams whose slots were taken over
        with torch.cuda.stream(s):
            c = torch.zeros(8, dtype=torch.int64, device="cuda")
            pp.pospopcnt(buf, 8, counters=c)
        outs.append((s, c))
    torch.cuda.synchronize()
    for s, c in outs:
        assert [int(x) for x in c.cpu()] == want
    for h, _ in streams + busy:
        rt.cudaStreamDestroy(h)


def test_direct_small_calls(cuda, oracle, rng):
    """Synchronous small calls take the direct path (pp_count_direct_kernel:
    one CTA reads the bytes in place -- host bytes through the pinned
    small-call buffer over the link -- and publishes counts + a flag in
    mapped pinned memory the host polls; ranges of several chunks: one CTA
    per chunk, the last one publishes).  Sizes around its chunk (32 KiB) and
    cut-off (512 KiB host, 16 MiB device) boundaries, every width, odd offsets, both entry
    points (pp_count_sync via list counters, pp_count_host via host bytes),
    accumulate semantics, and many calls back to back (the flag's sequence
    number must never let a call read its predecessor's counts)."""
    torch, pp = cuda
    K = 1 << 10
    data = rng.randbytes(16500 * K)
    host = np.frombuffer(data, np.uint8)
    buf = torch.from_numpy(host.copy()).cuda()
    sizes = [8, 64, 4 * K, 32 * K - 16, 32 * K, 32 * K + 16, 64 * K + 8, 128 * K - 8, 128 * K,
             128 * K + 8, 256 * K + 8,
             512 * K - 8, 512 * K, 512 * K + 8, 1024 * K + 8, 4096 * K + 64, 16384 * K - 8,
             16384 * K, 16384 * K + 8]
    for w in (8, 16, 32, 64):
        for n in sizes:
            for off in (0, 3, 13):
                want = oracle.hs512(host, off, n, w)
                assert pp.pospopcnt(pp.InputView(buf, off, n), w) == want, ("sync", w, n, off)
                assert pp.pospopcnt(data[off:off + n], w) == want, ("host", w, n, off)
    c = [5] * 16
    want = oracle.hs512(host, 1, 1000, 16)
    pp.pospopcnt(pp.InputView(buf, 1, 1000), 16, counters=c)
    pp.pospopcnt(data[1:1001], 16, counters=c)
    assert c == [5 + 2 * v for v in want]
    # back to back, alternating inputs: each call returns its own counts
    wants = [oracle.hs512(host, 64 * i, 512 + 8 * i, 8) for i in range(8)]
    for rep in range(300):
        i = rep % 8
        assert pp.pospopcnt(pp.InputView(buf, 64 * i, 512 + 8 * i), 8) == wants[i]
        assert pp.pospopcnt(data[64 * i:64 * i + 512 + 8 * i], 8) == wants[i]
    # a busy stream: the bounded poll gives way to a stream wait
    torch.cuda._sleep(int(1e8))  # ~50 ms of device time ahead of the count
    assert pp.pospopcnt(pp.InputView(buf, 64, 520), 8) == wants[1]
    # a second stream and a second thread have their own publish slots
    import threading
    errs = []

    def worker(k):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for rep in range(200):
                i = (rep + k) % 8
                if pp.pospopcnt(pp.InputView(buf, 64 * i, 512 + 8 * i), 8) != wants[i]:
                    errs.append((k, rep))
    ts = [threading.Thread(target=worker, args=(k,)) for k in range(3)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert not errs
