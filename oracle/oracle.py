"""CPU oracle for the positional population count — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  It is the checker, never the
thing measured as the product: paper_2412_16370_b200 never imports it.

Three independent codings of the reference's arithmetic:

* ``scalar``      -- C restatement of scalar_pospopcnt (core.py:82-96)
* ``hs512``       -- C restatement of the reference's fastest CPU path,
                     NumbaKernel.run + _nbkern.run_main (kernels.py:242-270,
                     _nbkern.py:43-177), optionally threaded over shards
* ``unpackbits``  -- numpy: np.unpackbits(..., bitorder="little") summed per
                     bit position (the survey's independent cross-check)

plus the byte-identical CPU twins of the device-side generators
(paper_2412_16370_b200/csrc/pp_gen.cu) and the bounded-Zipf thresholds of
config C3.  Parity of the C restatement is pinned against the reference
itself by the committed fixtures in tests/golden/ (tests/test_oracle.py).
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC_PATH = os.path.join(HERE, "pospopcnt_oracle.c")

_lib = None


def build(force=False):
    """Compile liboracle.so from pospopcnt_oracle.c (make, in this directory)."""
    stale = (not os.path.exists(LIB_PATH)
             or os.path.getmtime(SRC_PATH) > os.path.getmtime(LIB_PATH))
    if force or stale:
        subprocess.run(["make", "-s", "-C", HERE, "-B" if force else "liboracle.so"],
                       check=True, capture_output=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        u8p = ctypes.c_void_p
        sz = ctypes.c_size_t
        u64 = ctypes.c_uint64
        L.oracle_scalar.argtypes = [u8p, sz, ctypes.c_int, u8p]
        L.oracle_hs512.argtypes = [u8p, sz, sz, ctypes.c_int, u8p]
        L.oracle_hs512_mt.argtypes = [u8p, sz, sz, ctypes.c_int, u8p, ctypes.c_int]
        L.oracle_segments.argtypes = [u8p, u8p, sz, ctypes.c_int, u8p, ctypes.c_int]
        L.oracle_views.argtypes = [u8p, u8p, u8p, sz, ctypes.c_int, u8p, ctypes.c_int]
        L.oracle_gen_uniform.argtypes = [u8p, sz, u64, u64]
        L.oracle_gen_bernoulli.argtypes = [u8p, sz, u64, u64, ctypes.c_uint32]
        L.oracle_gen_blocks.argtypes = [u8p, sz, u64, u64, u64]
        L.oracle_gen_onehot32.argtypes = [u8p, sz, u64, u64, u8p]
        L.oracle_gen_codes8.argtypes = [u8p, sz, u64, u64, u8p]
        L.oracle_gen_codes8.restype = None
        L.oracle_block_q.argtypes = [u64, u64]
        L.oracle_block_q.restype = ctypes.c_uint32
        for f in (L.oracle_gen_uniform, L.oracle_gen_bernoulli, L.oracle_gen_blocks,
                  L.oracle_gen_onehot32):
            f.restype = None
        _lib = L
    return _lib


def _u8(data):
    """Contiguous uint8 numpy view of bytes-like data (no copy when possible)."""
    if isinstance(data, np.ndarray):
        return np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    return np.frombuffer(memoryview(data).cast("B"), dtype=np.uint8)


def _check(rc):
    if rc == 1:
        raise ValueError("word width must be one of (8, 16, 32, 64)")
    if rc == 2:
        raise ValueError("input length is not a multiple of the word size")
    if rc:
        raise RuntimeError(f"oracle failed with code {rc}")


def scalar(data, w):
    """scalar_pospopcnt (core.py:82-96) in C; returns a list of w ints."""
    a = _u8(data)
    out = np.zeros(64, dtype=np.uint64)
    _check(lib().oracle_scalar(a.ctypes.data, a.size, w, out.ctypes.data))
    return [int(x) for x in out[:w]]


def hs512(base, offset, nbytes, w, threads=1):
    """NumbaKernel.run(InputView(base, offset, nbytes), w) restated in C."""
    a = _u8(base)
    if offset < 0 or nbytes < 0 or offset + nbytes > a.size:
        raise ValueError("view extends past the end of its buffer")
    out = np.zeros(64, dtype=np.uint64)
    if threads > 1:
        rc = lib().oracle_hs512_mt(a.ctypes.data, offset, nbytes, w, out.ctypes.data, threads)
    else:
        rc = lib().oracle_hs512(a.ctypes.data, offset, nbytes, w, out.ctypes.data)
    _check(rc)
    return [int(x) for x in out[:w]]


def segments(base, offsets, w, threads=None):
    """Row s = NumbaKernel.run(InputView(base, offsets[s], offsets[s+1]-offsets[s]), w)."""
    a = _u8(base)
    offs = np.ascontiguousarray(offsets, dtype=np.uint64)
    nseg = offs.size - 1
    out = np.zeros((max(nseg, 0), w), dtype=np.uint64)
    if nseg <= 0:
        return out
    if offs.max() > a.size or (np.diff(offs.astype(np.int64)) < 0).any():
        raise ValueError("bad segment offsets")
    threads = threads or len(os.sched_getaffinity(0))
    _check(lib().oracle_segments(a.ctypes.data, offs.ctypes.data, nseg, w, out.ctypes.data,
                                 threads))
    return out


def views(base, starts, ends, w, threads=None):
    """Row s = NumbaKernel.run(InputView(base, starts[s], ends[s]-starts[s]), w)."""
    a = _u8(base)
    st = np.ascontiguousarray(starts, dtype=np.uint64)
    en = np.ascontiguousarray(ends, dtype=np.uint64)
    if st.shape != en.shape or (en < st).any() or (en.size and en.max() > a.size):
        raise ValueError("bad views")
    out = np.zeros((st.size, w), dtype=np.uint64)
    if st.size == 0:
        return out
    threads = threads or len(os.sched_getaffinity(0))
    _check(lib().oracle_views(a.ctypes.data, st.ctypes.data, en.ctypes.data, st.size, w,
                              out.ctypes.data, threads))
    return out


def unpackbits(data, w, chunk=1 << 24):
    """Independent numpy coding: per-position sums of little-endian bits."""
    a = _u8(data)
    step = w // 8
    if a.size % step:
        raise ValueError("input length is not a multiple of the word size")
    tot = np.zeros(w, dtype=np.int64)
    chunk -= chunk % step
    for s in range(0, a.size, chunk):
        bits = np.unpackbits(a[s:s + chunk], bitorder="little")
        tot += bits.reshape(-1, w).sum(axis=0, dtype=np.int64)
    return [int(x) for x in tot]


# ------------------------------------------------------------ generators

def gen_uniform(nbytes, seed, word_offset=0):
    assert nbytes % 8 == 0
    out = np.empty(nbytes // 8, dtype=np.uint64)
    lib().oracle_gen_uniform(out.ctypes.data, out.size, seed, word_offset)
    return out.view(np.uint8)


def gen_bernoulli(nbytes, seed, q, word_offset=0):
    assert nbytes % 8 == 0
    out = np.empty(nbytes // 8, dtype=np.uint64)
    lib().oracle_gen_bernoulli(out.ctypes.data, out.size, seed, word_offset, q)
    return out.view(np.uint8)


def gen_blocks(nbytes, seed, block_bytes=1 << 20, word_offset=0):
    assert nbytes % 8 == 0
    out = np.empty(nbytes // 8, dtype=np.uint64)
    lib().oracle_gen_blocks(out.ctypes.data, out.size, seed, word_offset, block_bytes)
    return out.view(np.uint8)


def block_q(seed, b):
    return int(lib().oracle_block_q(seed, b))


def zipf_thresholds(s=1.1, k=32):
    """Integer inverse-CDF thresholds of a bounded Zipf(s) on {1..k} (C3).

    thr[i] = round(2^32 * P(cat <= i)), i < k-1; a uniform u32 u maps to
    category #{i : thr[i] <= u} (0-based: bit position).
    """
    pmf = np.array([(i + 1) ** -s for i in range(k)], dtype=np.float64)
    pmf /= pmf.sum()
    cdf = np.cumsum(pmf)[:-1]
    thr = np.minimum(np.round(cdf * 2.0 ** 32), 2.0 ** 32 - 1).astype(np.uint32)
    return thr


def gen_onehot32(nbytes, seed, thr=None, word_offset=0):
    assert nbytes % 4 == 0
    thr = zipf_thresholds() if thr is None else np.ascontiguousarray(thr, dtype=np.uint32)
    out = np.empty(nbytes // 4, dtype=np.uint32)
    lib().oracle_gen_onehot32(out.ctypes.data, out.size, seed, word_offset, thr.ctypes.data)
    return out.view(np.uint8)


def gen_codes8(n, seed, thr=None, word_offset=0):
    thr = zipf_thresholds() if thr is None else np.ascontiguousarray(thr, dtype=np.uint32)
    out = np.empty(n, dtype=np.uint8)
    lib().oracle_gen_codes8(out.ctypes.data, out.size, seed, word_offset, thr.ctypes.data)
    return out


def categories(codes, w):
    """GROUP BY COUNT oracle: #{i : codes[i] == j} for j < w (== pospopcnt of one-hot words)."""
    c = np.asarray(codes).astype(np.int64).ravel()
    c = c[(c >= 0) & (c < w)]
    return [int(x) for x in np.bincount(c, minlength=w)[:w]]


def onehot_expected(nwords, seed, thr=None, word_offset=0):
    """Closed-form C3 oracle: counters[j] = #words whose one-hot bit is j."""
    thr = zipf_thresholds() if thr is None else thr
    words = gen_onehot32(nwords * 4, seed, thr, word_offset).view(np.uint32)
    cats = np.log2(words).astype(np.int64)
    return [int(x) for x in np.bincount(cats, minlength=32)]
