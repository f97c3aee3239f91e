"""Memory-safety evidence without compute-sanitizer (closed on this pool):
the PP_CHECK_BOUNDS=1 build of the library (libpospopcnt_b200_checked.so,
built in-tree by build()) checks, before issuing it, every global load and
bulk-copy source range against the caller's [data, data + nbytes) as the API
received it, every shared-memory stage index, every chunk id, and per launch
that the chunks consumed total the chunks issued (a skipped or repeated
mbarrier phase breaks that).  A failed check skips the access and is
recorded; pp_check_status reads the record.

Reference contract: nothing outside the buffer is read (edges.py:1-10,
pkg/tests/test_kernels.py:83-91).  The suites below -- exact-allocation
edges, the c1 sweep, segmented/ragged/tiny/batch arrays, the golden vectors
incl. 64 GiB C5, categories, the direct small-call path, and a 60 s
randomised soak -- run on the
checked build; every process reports its record at exit (PP_CHECK_REPORT)
and every record must be clean.  The negative test corrupts the launchers'
derived ranges on purpose and shows the checks fire.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _checked_lib():
    from paper_2412_16370_b200 import build
    lib = build.CHECKED_LIB
    if not os.path.exists(lib):
        build.build_checked()
    return lib


def _records(path):
    recs = []
    with open(path) as f:
        for ln in f:
            parts = ln.split()
            assert parts[1] != "error", ln
            recs.append({"pid": int(parts[0]), "checked": int(parts[1]), "fails": int(parts[2]),
                         "line": int(parts[3]), "addr": parts[4], "lo": parts[5],
                         "hi": parts[6]})
    return recs


def test_checked_build_suites_clean(cuda, tmp_path):
    lib = _checked_lib()
    report = tmp_path / "checks.txt"
    env = dict(os.environ, PP_LIB_PATH=lib, PP_CHECK_REPORT=str(report))
    res = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
         os.path.join(ROOT, "tests", "test_gpu_edges.py"),
         os.path.join(ROOT, "tests", "test_gpu_golden.py"),
         os.path.join(ROOT, "tests", "test_gpu_segmented.py"),
         os.path.join(ROOT, "tests", "test_gpu_categories.py"),
         os.path.join(ROOT, "tests", "test_gpu_parity.py") + "::test_direct_small_calls"],
        capture_output=True, text=True, timeout=1500, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-2000:]
    res = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "fuzz.py"),
                          "--seconds", "60", "--threads", "3", "--seed", "11"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert res.returncode == 0 and "failures: []" in res.stdout, \
        res.stdout[-3000:] + res.stderr[-3000:]
    recs = _records(report)
    # pytest itself, scripts/sanitize_cases.py and the fuzz soak at least
    assert len(recs) >= 3, recs
    assert all(r["checked"] == 1 for r in recs), recs  # the checked build was loaded
    assert all(r["fails"] == 0 for r in recs), [r for r in recs if r["fails"]]


_NEG = r"""
import sys, torch
sys.path.insert(0, %(root)r)
from paper_2412_16370_b200 import _lib
import paper_2412_16370_b200 as pp
lib = _lib.load()
assert _lib.check_status(reset=True)["checked_build"]
n = (40 << 20) + 24                     # > 1 chunk, misaligned tail
buf = torch.full((n + 3,), 0xA5, dtype=torch.uint8, device="cuda")
view = pp.InputView(buf, 3, n)
def count():
    c = torch.zeros(64, dtype=torch.int64, device="cuda")
    pp.pospopcnt(view, 8, counters=c)
    torch.cuda.synchronize()
    return c
want = count()
assert _lib.check_status()["fails"] == 0
out = []
for mode in (1, 2):
    _lib.check(lib.pp_debug_corrupt(mode))
    count()
    _lib.check(lib.pp_debug_corrupt(0))
    st = _lib.check_status(reset=True)
    out.append((mode, st["fails"], st["first_line"]))
# segmented, fixed segments: the TMA ring (4 KiB), the LDG kernel (>= 8 KiB
# hint) and the one-lane kernel (64 B)
seg = torch.full((80 << 20,), 0x5A, dtype=torch.uint8, device="cuda")
for sb, nseg, lanes in ((4096, 16384, None), (8192, 1024, 8), (64, 1024, None)):
    _lib.check(lib.pp_debug_corrupt(3))
    pp.pospopcnt_fixed(seg[16:16 + sb * nseg], sb, 64, lanes=lanes)
    torch.cuda.synchronize()
    _lib.check(lib.pp_debug_corrupt(0))
    st = _lib.check_status(reset=True)
    out.append((3, st["fails"], st["first_line"]))
assert torch.equal(count(), want) and _lib.check_status()["fails"] == 0
print("NEG", out)
"""


def test_checks_fire_on_corrupted_ranges(cuda):
    """Corrupted launch ranges are caught: every mode records failed checks
    (and, since the checks skip the access, nothing is read out of range and
    the context stays usable: the clean count afterwards is exact)."""
    lib = _checked_lib()
    env = dict(os.environ, PP_LIB_PATH=lib)
    res = subprocess.run([sys.executable, "-c", _NEG % {"root": ROOT}], capture_output=True,
                         text=True, timeout=600, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    line = [ln for ln in res.stdout.splitlines() if ln.startswith("NEG")][0]
    cases = eval(line[4:])  # noqa: S307 - our own printed list of tuples
    assert len(cases) == 5 and all(fails > 0 and first_line > 0 for _, fails, first_line in cases), \
        cases


def test_unchecked_build_reports_unchecked(cuda):
    from paper_2412_16370_b200 import _lib
    st = _lib.check_status()
    assert not st["checked_build"] and st["fails"] == 0
    assert _lib.load().pp_debug_corrupt(1) == _lib.PP_EARG
