"""Pin the CPU oracle to the reference itself (runs without a GPU).

tests/golden/golden.json holds counters computed by the REFERENCE package
(/root/reference, numba + numpy + scalar kernels) on seeded generator inputs,
written by tests/golden/make_golden.py.  Here the C restatement (oracle/) and
the independent numpy coding must reproduce every one of them bit-exactly,
and the generator twins must reproduce every recorded input hash.
"""

import hashlib
import json
import os
import random

import numpy as np
import pytest

from conftest import oracle_bits

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.json")
MIB = 1 << 20


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def _gen(O, spec):
    kind, n, seed, off = spec["kind"], spec["nbytes"], spec["seed"], spec.get("word_offset", 0)
    if kind == "uniform":
        return O.gen_uniform(n, seed, off)
    if kind == "bernoulli":
        return O.gen_bernoulli(n, seed, spec["q"], off)
    if kind == "blocks":
        return O.gen_blocks(n, seed, spec.get("block_bytes", MIB), off)
    return O.gen_onehot32(n, seed, word_offset=off)


def test_known_answers(golden, oracle):
    assert len(golden["known_answers"]) >= 10
    for ka in golden["known_answers"]:
        w = ka["w"]
        if "hex" in ka:
            data = bytes.fromhex(ka["hex"])
        elif "repeat_hex" in ka:
            data = bytes.fromhex(ka["repeat_hex"]) * ka["repeat"]
        else:
            data = bytes(ka["zeros"])
        assert oracle.scalar(data, w) == ka["expected"], ka["source"]
        assert oracle.hs512(data, 0, len(data), w) == ka["expected"], ka["source"]
        assert oracle.unpackbits(data, w) == ka["expected"], ka["source"]
        if len(data) < 5000:
            assert oracle_bits(data, w) == ka["expected"]


def _cases(golden, small):
    out = []
    for c in golden["cases"]:
        if (c["gen"]["nbytes"] <= 2 * MIB) == small:
            out.append(c)
    return out


def test_generated_cases_small(golden, oracle):
    cases = _cases(golden, True)
    assert len(cases) >= 30
    cache = {}
    for c in cases:
        key = json.dumps(c["gen"], sort_keys=True)
        if key not in cache:
            arr = _gen(oracle, c["gen"])
            assert hashlib.sha256(arr.tobytes()).hexdigest() == c["sha256"], c["name"]
            cache = {key: arr}
        arr = cache[key]
        got = oracle.hs512(arr, c["offset"], c["nbytes"], c["w"])
        assert got == c["numba"], c["name"]
        if "numpy" in c:
            assert c["numpy"] == c["numba"], c["name"]  # the reference agrees with itself
        if "scalar" in c:
            assert got == c["scalar"], c["name"]
            view = arr[c["offset"]:c["offset"] + c["nbytes"]]
            assert oracle.scalar(view, c["w"]) == c["scalar"], c["name"]
        view = arr[c["offset"]:c["offset"] + c["nbytes"]]
        assert oracle.unpackbits(view, c["w"]) == c["numba"], c["name"]


def test_generated_cases_full_size(golden, oracle):
    """C2 (1 GiB), C3 (4 GiB), C4 (64 MiB), C5 shard (1 GiB), all-ones: the oracle
    reproduces the reference's counters and the generators its input hashes."""
    cases = _cases(golden, False)
    names = {c["name"] for c in cases}
    assert {"c2_w8_1gib", "c3_w32_onehot_4gib", "c5_w16_shard3_1gib",
            "allones_w16_256mib"} <= names
    cache = {}
    threads = min(16, len(os.sched_getaffinity(0)))
    for c in cases:
        key = json.dumps(c["gen"], sort_keys=True)
        if key not in cache:
            cache.clear()
            arr = _gen(oracle, c["gen"])
            assert hashlib.sha256(arr.tobytes()).hexdigest() == c["sha256"], c["name"]
            cache[key] = arr
        arr = cache[key]
        got = oracle.hs512(arr, c["offset"], c["nbytes"], c["w"], threads=threads)
        assert got == c["numba"], c["name"]
        if "numpy" in c:
            assert c["numpy"] == c["numba"]
    cache.clear()


def test_c1_sweep_digest(golden, oracle):
    """acceptance c1: all (alignment, length, width) views; digest of the
    reference's outputs must match the oracle's row for row."""
    base = np.frombuffer(random.Random(20240).randbytes(64 + 4096), np.uint8)
    for w in (8, 16, 32, 64):
        lens = np.arange(0, 4097, w // 8, dtype=np.uint64)
        starts = np.repeat(np.arange(64, dtype=np.uint64), lens.size)
        ends = starts + np.tile(lens, 64)
        rows = oracle.views(base, starts, ends, w)
        dig = golden["digests"][f"c1_sweep_w{w}"]
        assert rows.shape[0] == dig["rows"]
        assert hashlib.sha256(np.ascontiguousarray(rows).tobytes()).hexdigest() == \
            dig["sha256_u64_rows"], w


def test_c4_segmented_digest(golden, oracle):
    dig = golden["digests"]["c4_segmented_262144x4k_w64"]
    arr = _gen(oracle, dig["gen"])
    assert hashlib.sha256(arr.tobytes()).hexdigest() == dig["sha256"]
    offs = np.arange(262_145, dtype=np.uint64) * 4096
    rows = oracle.segments(arr, offs, 64)
    assert rows[0].tolist() == dig["row0"]
    assert rows.sum(axis=0).tolist() == dig["col_sums"]
    assert hashlib.sha256(np.ascontiguousarray(rows).tobytes()).hexdigest() == \
        dig["sha256_u64_rows"]


def test_oracle_codings_agree_random(oracle):
    """scalar == hs512 == unpackbits == bit-string coding on random views,
    including the 15-vector (960 B) short/main threshold straddles."""
    rng = random.Random(7)
    for case in range(400):
        w = (8, 16, 32, 64)[case % 4]
        step = w // 8
        n = rng.choice((0, step, 952, 960, 968, 1016, 1024, 1032, rng.randrange(0, 6000)))
        n -= n % step
        off = rng.randrange(0, 70)
        base = rng.randbytes(off + n + rng.randrange(0, 9))
        view = base[off:off + n]
        want = oracle.scalar(view, w)
        assert oracle.hs512(base, off, n, w) == want, (w, n, off)
        assert oracle.unpackbits(view, w) == want
        if n < 800:
            assert oracle_bits(view, w) == want


def test_oracle_threaded_equals_single(oracle):
    data = oracle.gen_uniform(64 * MIB, 3)
    one = oracle.hs512(data, 5, 64 * MIB - 8, 16)
    assert oracle.hs512(data, 5, 64 * MIB - 8, 16, threads=7) == one


def test_oracle_errors(oracle):
    with pytest.raises(ValueError):
        oracle.scalar(b"\x00" * 3, 16)
    with pytest.raises(ValueError):
        oracle.hs512(b"\x00" * 8, 0, 8, 12)
    with pytest.raises(ValueError):
        oracle.hs512(b"\x00" * 8, 4, 8, 8)


def test_onehot_closed_form(oracle):
    n = 1 << 20
    arr = oracle.gen_onehot32(4 * n, 0xC3)
    assert oracle.onehot_expected(n, 0xC3) == oracle.hs512(arr, 0, 4 * n, 32)
    words = arr.view(np.uint32)
    assert ((words & (words - 1)) == 0).all() and (words != 0).all()


def test_generator_statistics(oracle):
    b = oracle.gen_bernoulli(1 << 22, 11, 655)
    p = np.unpackbits(b).mean()
    assert abs(p - 655 / 65536) < 0.0005
    assert (oracle.gen_bernoulli(4096, 1, 65536) == 0xFF).all()
    assert (oracle.gen_bernoulli(4096, 1, 0) == 0).all()
    u = oracle.gen_uniform(1 << 22, 5)
    assert abs(np.unpackbits(u).mean() - 0.5) < 0.001
