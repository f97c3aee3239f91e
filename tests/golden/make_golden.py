#!/usr/bin/env python3
"""Generate tests/golden/golden.json by running the REFERENCE implementation.

Runs only in the build container, where /root/reference exists (it does not
exist on the GPU box; the committed JSON travels instead).  The reference
package is imported read-only under the alias ``pospopcnt_ref`` with numba's
cache redirected outside the reference tree (SURVEY.md section 8c gotchas).

Inputs come from the seeded generators (CPU twin in oracle/, byte-identical
to the device generators); each case records the generator spec, the sha256
of the generated buffer, and the counters the reference computes:

* ``numba``   -- get_kernel("numba").run(...)   (kernels.py:218-270), the
                 reference's fastest path, on every case
* ``numpy``   -- the default-dispatch kernel (kernels.py:178-215) where cheap
* ``scalar``  -- scalar_pospopcnt (core.py:82-96) on small cases

plus the inline known answers of the reference's tests, and sha256 digests of
the whole acceptance-c1 sweep and of the 262,144-row C4 segmented batch.

Usage: python tests/golden/make_golden.py [--full]   (--full adds the 64 GiB C5 total)
"""

import hashlib
import importlib.util
import json
import os
import random
import sys
import time
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
REF_SRC = os.environ.get("POSPOPCNT_REF_SRC", "/root/reference/pkg/src")

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/pospopcnt_ref_numba_cache")
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402

MIB = 1 << 20
GIB = 1 << 30


def load_reference():
    pkg_dir = os.path.join(REF_SRC, "pospopcnt")
    spec = importlib.util.spec_from_file_location(
        "pospopcnt_ref", os.path.join(pkg_dir, "__init__.py"),
        submodule_search_locations=[pkg_dir])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["pospopcnt_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def gen(spec):
    kind = spec["kind"]
    n, seed, off = spec["nbytes"], spec["seed"], spec.get("word_offset", 0)
    if kind == "uniform":
        return O.gen_uniform(n, seed, off)
    if kind == "bernoulli":
        return O.gen_bernoulli(n, seed, spec["q"], off)
    if kind == "blocks":
        return O.gen_blocks(n, seed, spec.get("block_bytes", MIB), off)
    if kind == "onehot32":
        return O.gen_onehot32(n, seed, word_offset=off)
    raise ValueError(kind)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _c5_part(i):
    ref = load_reference()
    spec = {"kind": "blocks", "nbytes": GIB, "seed": 0xC5, "word_offset": i * (GIB // 8)}
    data = gen(spec)
    k = ref.get_kernel("numba")
    return k.run(ref.InputView(data.tobytes(), 0, GIB), 16, [0] * 16), sha(data)


def main(full=False):
    ref = load_reference()
    numba_k = ref.get_kernel("numba")
    numpy_k = ref.get_kernel("numpy")
    IV = ref.InputView
    out = {"reference": REF_SRC, "generated_by": "tests/golden/make_golden.py",
           "known_answers": [], "cases": [], "digests": {}}

    # --- inline known answers of the reference's own tests
    ka = [
        ("01 80", 16, "__init__.py:3-5"),
        ("ff ff", 16, "pkg/tests/test_core.py:14-15"),
        ("ff 00 81", 8, "pkg/tests/test_edges.py:100-103"),
        ("0f", 8, "pkg/tests/test_cli.py:42-47"),
        ("", 8, "pkg/tests/test_core.py:18-20"),
        ("", 64, "pkg/tests/test_core.py:18-20"),
    ]
    for hx, w, src in ka:
        data = bytes.fromhex(hx)
        out["known_answers"].append({"hex": hx, "w": w, "source": src,
                                     "expected": ref.pospopcnt(data, w)})
    for n in (1, 1000, 1_000_000):
        data = b"\x01\x80" * n
        out["known_answers"].append({"repeat_hex": "0180", "repeat": n, "w": 16,
                                     "source": "pkg/tests/test_kernels.py:32-37",
                                     "expected": numba_k.run(IV.of(data), 16, [0] * 16)})
    data = bytes(16 * 1024)
    out["known_answers"].append({"zeros": 16 * 1024, "w": 16,
                                 "source": "pkg/tests/test_kernels.py:26-29",
                                 "expected": numba_k.run(IV.of(data), 16, [0] * 16)})

    # --- seeded generator cases
    cases = []
    for w in (8, 16, 32, 64):
        for n, off in ((0, 0), (8, 1), (120, 3), (960, 0), (961 * 8 // 8 * 8, 7), (4096, 5),
                       (65536, 9), (1 << 20, 13)):
            cases.append((f"uniform_w{w}_n{n}_off{off}",
                          {"kind": "uniform", "nbytes": (1 << 20) + 64, "seed": 0x600D + w},
                          off, n - n % (w // 8), w))
    cases.append(("c1_w16_2mib", {"kind": "uniform", "nbytes": 2 * MIB, "seed": 0xC1}, 0,
                  2 * MIB, 16))
    cases.append(("c2_w8_1gib", {"kind": "uniform", "nbytes": GIB, "seed": 0xC2}, 0, GIB, 8))
    cases.append(("c3_w32_onehot_4gib", {"kind": "onehot32", "nbytes": 4 * GIB, "seed": 0xC3},
                  0, 4 * GIB, 32))
    c4spec = {"kind": "bernoulli", "nbytes": 64 * MIB + 64, "seed": 0xC4, "q": 655}
    for n in (1, 3, 17, 255, 512, 8192, 131072, 8388608):
        for off in range(1, 8):
            cases.append((f"c4_w64_n{n}_off{off}", c4spec, off, 8 * n, 64))
    cases.append(("c5_w16_shard3_1gib", {"kind": "blocks", "nbytes": GIB, "seed": 0xC5,
                                         "word_offset": 3 * (GIB // 8)}, 0, GIB, 16))
    cases.append(("allones_w16_256mib", {"kind": "bernoulli", "nbytes": 256 * MIB, "seed": 1,
                                         "q": 65536}, 0, 256 * MIB, 16))

    cache = {}
    for name, spec, off, n, w in cases:
        key = json.dumps(spec, sort_keys=True)
        if key not in cache:
            cache.clear()
            t = time.time()
            arr = gen(spec)
            cache[key] = (arr, arr.tobytes(), sha(arr))
            print(f"gen {spec} {time.time() - t:.1f}s", flush=True)
        arr, raw, digest = cache[key]
        view = IV(raw, off, n)
        t = time.time()
        rec = {"name": name, "gen": spec, "offset": off, "nbytes": n, "w": w,
               "sha256": digest, "numba": numba_k.run(view, w, [0] * w)}
        if n <= 64 * MIB:
            rec["numpy"] = numpy_k.run(view, w, [0] * w)
        if n <= 65536:
            rec["scalar"] = ref.scalar_pospopcnt(view, w)
        out["cases"].append(rec)
        print(f"{name}: {time.time() - t:.2f}s", flush=True)
    cache.clear()

    # --- acceptance c1 sweep digest (pkg/tests/test_acceptance.py:41-64)
    base = random.Random(20240).randbytes(64 + 4096)
    for w in (8, 16, 32, 64):
        t = time.time()
        rows = []
        for a in range(64):
            for n in range(0, 4097, w // 8):
                rows.append(numba_k.run(IV(base, a, n), w, [0] * w))
        arr = np.array(rows, dtype=np.uint64)
        out["digests"][f"c1_sweep_w{w}"] = {
            "sha256_u64_rows": sha(arr), "rows": len(rows),
            "order": "a in 0..63 (outer), n in 0..4096 step w/8 (inner)",
            "base": "random.Random(20240).randbytes(64 + 4096)"}
        print(f"c1 sweep w={w}: {time.time() - t:.1f}s", flush=True)

    # --- C4 segmented batch digest: 262,144 x 4 KiB, w=64
    spec = {"kind": "bernoulli", "nbytes": GIB, "seed": 0xC4 + 1, "q": 655}
    t = time.time()
    arr = gen(spec)
    raw = arr.tobytes()
    rows = np.empty((262_144, 64), dtype=np.uint64)
    for s in range(262_144):
        rows[s] = numba_k.run(IV(raw, 4096 * s, 4096), 64, [0] * 64)
    out["digests"]["c4_segmented_262144x4k_w64"] = {
        "gen": spec, "sha256": sha(arr), "sha256_u64_rows": sha(rows),
        "row0": rows[0].tolist(), "col_sums": rows.sum(axis=0).tolist()}
    print(f"c4 segmented: {time.time() - t:.1f}s", flush=True)
    del raw, arr

    if full:
        t = time.time()
        tot = [0] * 16
        with ProcessPoolExecutor(8) as ex:
            parts = list(ex.map(_c5_part, range(64)))
        for c, _ in parts:
            tot = [x + y for x, y in zip(tot, c)]
        out["digests"]["c5_w16_64gib_total"] = {
            "gen": {"kind": "blocks", "nbytes": 64 * GIB, "seed": 0xC5},
            "expected": tot, "part_sha256": [s for _, s in parts]}
        print(f"c5 64 GiB: {time.time() - t:.1f}s", flush=True)

    path = os.path.join(HERE, "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main(full="--full" in sys.argv)
