"""GPU parity of the fused one-hot producer (pospopcnt_categories).

Contract: pospopcnt_categories(codes, w) == pospopcnt(one_hot_w(codes), w)
== bincount of the codes below w.  Pinned to the reference through config
C3: the u8 codes generated with C3's draws must reproduce the reference's own
counters of the 4 GiB one-hot array (tests/golden/golden.json).
"""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.json")


def test_c3_codes_equal_reference_onehot_counts(cuda):
    torch, pp = cuda
    from paper_2412_16370_b200 import gen
    with open(GOLDEN) as f:
        case = {c["name"]: c for c in json.load(f)["cases"]}["c3_w32_onehot_4gib"]
    codes = gen.generate("codes8", 1 << 30, 0xC3)  # 2^30 codes, one per byte
    assert pp.pospopcnt_categories(codes, 32) == case["numba"]
    # back to back with input_ready (the codes are written once, before):
    # every width's counts, accumulated on the device, still the reference's
    cnt = torch.zeros((3, 32), dtype=torch.int64, device="cuda")
    for r in range(3):
        pp.pospopcnt_categories(codes, 32, counters=cnt[r], input_ready=True)
        pp.pospopcnt_categories(codes, 32, counters=cnt[r], input_ready=True)
    for r in range(3):
        assert [int(x) for x in cnt[r].cpu()] == [2 * v for v in case["numba"]], r
    onehot = gen.generate("onehot32", 4 << 30, 0xC3)
    assert pp.pospopcnt(onehot, 32) == case["numba"]
    del codes, onehot
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dtype", ("uint8", "int16", "int32"))
def test_random_codes_vs_oracle_and_materialised_onehot(cuda, oracle, dtype):
    torch, pp = cuda
    rng = np.random.default_rng(7)
    tdt = {"uint8": torch.uint8, "int16": torch.int16, "int32": torch.int32}[dtype]
    for n in (0, 1, 15, 16, 17, 1000, 65536 + 7, 3_000_001):
        hi = 80 if dtype == "uint8" else 200  # some codes >= w: not counted
        host = rng.integers(0, hi, n).astype(dtype)
        full = torch.from_numpy(np.concatenate([np.zeros(3, dtype), host])).cuda()
        codes = full[3:]  # start 3 codes into the allocation (unaligned to 16 B)
        for w in (8, 16, 32, 64):
            want = oracle.categories(host, w)
            assert pp.pospopcnt_categories(codes, w) == want, (dtype, n, w)
            if n and n <= 65536 + 7 and w in (16, 64):
                oh = np.where(host.astype(np.int64) < w,
                              np.left_shift(np.uint64(1), np.minimum(host, w - 1).astype(np.uint64)),
                              np.uint64(0))
                words = oh.astype({16: np.uint16, 64: np.uint64}[w])
                assert pp.pospopcnt(torch.from_numpy(words.view(np.uint8)).cuda(), w) == want
    c = torch.ones(32, dtype=torch.int64, device="cuda")
    codes = torch.from_numpy(rng.integers(0, 32, 10_000).astype(np.uint8)).cuda()
    pp.pospopcnt_categories(codes, 32, counters=c)
    want = oracle.categories(codes.cpu().numpy(), 32)
    assert [int(x) for x in c.cpu()] == [v + 1 for v in want]


def test_every_u8_code_at_every_byte_position(cuda, oracle):
    """All 256 code values in every byte lane of the 16-byte vectors (the
    one-hot expansion works on packed bytes: codes >= w, >= 128 and the
    boundary codes w-1, w, 7, 8, 127, 128, 255 must all be exact), mixed into
    uniform random codes so that vectors with and without large codes occur."""
    torch, pp = cuda
    rng = np.random.default_rng(99)
    base = np.arange(256, dtype=np.uint8)
    # 17 shifted copies: code v sits at byte position (v + k) mod 16 for every k
    ex = np.concatenate([np.roll(base, k) for k in range(17)])
    small = rng.integers(0, 8, 1 << 16).astype(np.uint8)        # vectors of valid codes only
    uni = rng.integers(0, 256, (1 << 22) + 9).astype(np.uint8)
    for host in (ex, np.concatenate([small, ex, uni, small])):
        codes = torch.from_numpy(host).cuda()
        for w in (8, 16, 32, 64):
            assert pp.pospopcnt_categories(codes, w) == oracle.categories(host, w), (w, host.size)


@pytest.mark.parametrize("w", (16, 32))
def test_small_code_fast_path_mixed_with_exact_path(cuda, oracle, w):
    """w = 32 takes a fast expansion when a warp's 8 vectors hold only codes
    < 32 (shift amounts taken mod 32, bytes brought down by mul.hi); w = 16
    runs the same inputs through the exact path.  Every code < w, then the
    same with one out-of-range code (w, 255, or a value whose low 5 bits
    alias a valid code) planted in every 7th 4 KiB block, so warps of one
    launch switch between the two paths; and the partial last chunk."""
    torch, pp = cuda
    rng = np.random.default_rng(1000 + w)
    n = (48 << 20) + 4099
    host = rng.integers(0, w, n).astype(np.uint8)
    codes = torch.from_numpy(host).cuda()
    assert pp.pospopcnt_categories(codes, w) == oracle.categories(host, w)
    mixed = host.copy()
    bad = np.array([w, 255, w + 1, 32 + 3, 64 + 5, 128], dtype=np.uint8)
    pos = np.arange(0, n, 7 * 4096) + rng.integers(0, 4096, (n + 7 * 4096 - 1) // (7 * 4096))
    pos = pos[pos < n]
    mixed[pos] = bad[np.arange(pos.size) % bad.size]
    codes = torch.from_numpy(mixed).cuda()
    assert pp.pospopcnt_categories(codes, w) == oracle.categories(mixed, w)
    for m in (1, 15, 16 * 1024 + 3, (1 << 20) - 1):  # short, and partial last chunks
        assert pp.pospopcnt_categories(codes[:m], w) == oracle.categories(mixed[:m], w), m
    shifted = torch.from_numpy(np.concatenate([np.zeros(5, np.uint8), host])).cuda()[5:]
    assert pp.pospopcnt_categories(shifted, w) == oracle.categories(host, w)


@pytest.mark.parametrize("dtype", ("int16", "uint16", "int32", "uint32"))
def test_wide_codes_boundaries_every_lane(cuda, oracle, dtype):
    """2- and 4-byte codes on the one-hot TMA path: boundary values (w - 1,
    w, 7, 8, 15, 16, 31, 32, 63, 64, the type's max, negatives) in every
    code slot of the 16-byte vectors, mixed with uniform codes, partial
    chunks and an unaligned (but code-aligned) start."""
    torch, pp = cuda
    rng = np.random.default_rng(123)
    info = np.iinfo(dtype)
    special = np.array([0, 1, 7, 8, 15, 16, 31, 32, 63, 64, 65, 255, 256, 1000,
                        info.max, info.max - 1] + ([-1, -2, info.min] if info.min < 0 else []),
                       dtype=np.int64).astype(dtype)
    per_vec = 16 // np.dtype(dtype).itemsize
    ex = np.concatenate([np.roll(special, k) for k in range(per_vec + 1)])
    small = rng.integers(0, 8, 4099).astype(dtype)
    uni = rng.integers(0, 80, (1 << 21) + 5).astype(dtype)
    host = np.concatenate([ex, small, uni, ex])
    aligned = torch.from_numpy(host.copy()).cuda()
    shifted = torch.from_numpy(np.concatenate([np.zeros(3, dtype), host])).cuda()[3:]
    for codes in (aligned, shifted, aligned[: ex.size + 5]):
        want = host[: codes.numel()]
        for w in (8, 16, 32, 64):
            assert pp.pospopcnt_categories(codes, w) == oracle.categories(want, w), (w, codes.numel())


def test_one_bin_past_2_32(cuda):
    """Every code in one bin, 10 GiB of them: that counter passes 2^32 (u64
    all the way; on the PP_CAT_PATH=smem alternative each thread's u16 column
    sits at its 65535 limit and the launch is split)."""
    torch, pp = cuda
    n = (10 << 30) + 5
    codes = torch.full((n,), 7, dtype=torch.uint8, device="cuda")
    got = pp.pospopcnt_categories(codes, 8)
    assert got == [0] * 7 + [n]
    del codes
    torch.cuda.empty_cache()


def test_errors(cuda):
    torch, pp = cuda
    with pytest.raises(ValueError):
        pp.pospopcnt_categories(torch.zeros(4, dtype=torch.float32, device="cuda"), 8)
    with pytest.raises(ValueError):
        pp.pospopcnt_categories(torch.zeros(4, dtype=torch.uint8, device="cuda"), 12)
    with pytest.raises(ValueError):
        pp.pospopcnt_categories(torch.zeros(4, dtype=torch.uint8, device="cuda"), 16,
                                counters=[0] * 8)


def test_histogram_alternative_path(cuda):
    """PP_CAT_PATH=smem (the shared-memory histogram, kept for A/B runs) must
    stay exact too; the path is chosen once per process, so in a child."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    child = (
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {root!r})\n"
        "from oracle import oracle as O\n"
        "import paper_2412_16370_b200 as pp\n"
        "rng = np.random.default_rng(5)\n"
        "for dt in ('uint8', 'int16', 'int32'):\n"
        "    host = rng.integers(-3 if dt != 'uint8' else 0, 90, 3_000_017).astype(dt)\n"
        "    codes = torch.from_numpy(host).cuda()\n"
        "    for w in (8, 16, 32, 64):\n"
        "        assert pp.pospopcnt_categories(codes, w) == O.categories(host, w), (dt, w)\n"
        "print('ok')\n")
    env = dict(os.environ, PP_CAT_PATH="smem")
    res = subprocess.run([sys.executable, "-c", child], env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0 and res.stdout.strip().endswith("ok"), res.stdout + res.stderr
