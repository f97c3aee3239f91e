"""SURVEY.md 8f item 1 on hardware: the reference's own dispatch, test
suite, selftest and benchmark harness drive the b200 kernel on a B200.

The unmodified reference is installed under baseline/_ref (with its test
suite staged beside it) by scripts/stage_reference.sh in the build
container; that directory travels to the GPU box (git-ignored, not
gpurun-ignored).  /root/reference is never read here.  Every reference
interface is reached through ``ref_plugin.register`` only.
"""

import io
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "pkg_tests")


def _env(**extra):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests")])
    env.update(PP_REF_DIR=REF, NUMBA_CACHE_DIR="/tmp/pp_numba_cache",
               PYTHONDONTWRITEBYTECODE="1", **extra)
    return env


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "pospopcnt")) or not os.path.isdir(REF_TESTS):
        # build() stages it wherever /root/reference exists; a skip (not a
        # failure) keeps `pytest -x` running the rest of the GPU suite
        pytest.skip("baseline/_ref (the installed reference + its tests) is missing: "
                    "__graft_entry__.build() / scripts/stage_reference.sh stage it")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import pospopcnt
    assert os.path.abspath(pospopcnt.__file__).startswith(REF), pospopcnt.__file__
    from paper_2412_16370_b200 import ref_plugin
    k = ref_plugin.register(pospopcnt)
    assert k.available()
    return pospopcnt, k


def _pytest(args, **env):
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "refsuite_plugin", "-p",
           "no:cacheprovider", "-c", os.devnull, "--rootdir", REF_TESTS, *args]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=REF_TESTS,
                         env=_env(**env))
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-2000:]
    return res.stdout


def test_reference_suite_with_b200_registered(ref):
    """The reference's own tests (pkg/tests: kernels, core, edges, cli, bench,
    acceptance criteria 2-7, ...) with b200 in the registry: every
    kernel-parametrised test includes b200 next to portable/int256/numba/
    numpy, and the registry/CLI/bench contracts still hold with it added.
    Criterion 1 runs on its own below (b200 only)."""
    # test_instrumented_modes_match_default (test_kernels.py:135-142) exempts
    # the compiled kernel by NAME ("numba"); b200 is compiled too and, per the
    # same contract (kernels.py:243-244), rejects fa=/probe= -- asserted below
    out = _pytest(["-k", "not criterion_1 and not test_instrumented_modes_match_default"])
    assert "passed" in out and "failed" not in out


def test_b200_rejects_instrumentation_like_numba(ref):
    """test_numba_rejects_instrumentation (test_kernels.py:145-150), for b200."""
    P, k = ref
    from pospopcnt.csa import full_adder
    for kern in (k, P.get_kernel("numba")):
        with pytest.raises(ValueError):
            kern.run(P.InputView.of(b"\x00" * 16), 8, [0] * 8, fa=full_adder)
        with pytest.raises(ValueError):
            kern.run(P.InputView.of(b"\x00" * 16), 8, [0] * 8, probe=lambda st: None)


def test_reference_criterion1_sweep_on_b200(ref):
    """Criterion 1 (pkg/tests/test_acceptance.py:41-64): 491,776 kernel calls
    (every length 0..4096 at every offset 0..63, w = 8/16/32/64) against the
    running scalar oracle -- with b200 as the only available kernel."""
    out = _pytest(["test_acceptance.py::test_criterion_1_oracle_equivalence_sweep", "-s"],
                  PP_REF_ONLY_B200="1")
    assert "491776 kernel calls over 1 kernels" in out, out[-2000:]


def test_reference_dispatch_reaches_b200(ref):
    """pospopcnt() / get_kernel / select_kernel / POSPOPCNT_KERNEL
    (kernels.py:293-333) resolve to the registered b200 kernel."""
    P, k = ref
    assert P.get_kernel("b200") is k
    assert P.select_kernel("b200") is k
    assert "b200" in [d.name for d, ok in P.list_kernels() if ok]
    data = bytes(range(256)) * 4099
    want = P.pospopcnt(data, 16, kernel="numba")
    assert P.pospopcnt(data, 16, kernel="b200") == want
    assert P.pospopcnt(P.InputView(data, 5, 8000), 64, kernel=k) == \
        P.scalar_pospopcnt(P.InputView(data, 5, 8000), 64)
    os.environ[P.kernels.KERNEL_ENV] = "b200"
    try:
        assert P.select_kernel() is k
        assert P.pospopcnt(data, 8) == P.pospopcnt(data, 8, kernel="numba")
    finally:
        del os.environ[P.kernels.KERNEL_ENV]


def test_reference_selftest_drives_b200(ref):
    """selftest.run_selftest (selftest.py:44-90): 1000 fuzz cases against
    the scalar oracle / a second kernel, b200 alone and b200 + numba."""
    P, k = ref
    from pospopcnt import selftest
    lines = []
    assert selftest.run_selftest(iterations=1000, seed=7, kernels=[k], out=lines.append), lines
    assert selftest.run_selftest(iterations=400, seed=8,
                                 kernels=[k, P.get_kernel("numba")], out=lines.append), lines
    assert all("PASS" in ln for ln in lines)


def test_reference_cli_with_b200(ref, tmp_path):
    """The reference CLI (cli.py) with b200 registered: `count --kernel b200`,
    `kernels` listing, `selftest`, `bench --kernels b200,numba,baseline`."""
    f = tmp_path / "in.bin"
    f.write_bytes(bytes(range(256)) * 1000 + b"\x0f")
    code = (
        "import sys, pospopcnt\n"
        "from paper_2412_16370_b200 import ref_plugin\n"
        "ref_plugin.register(pospopcnt)\n"
        "from pospopcnt.cli import main\n"
        "sys.exit(main(sys.argv[1:]))\n")

    def cli(*args):
        res = subprocess.run([sys.executable, "-c", code, *args], capture_output=True,
                             text=True, timeout=600, env=_env())
        return res.returncode, res.stdout, res.stderr

    rc, out_b, err = cli("count", "--kernel", "b200", "--width", "8", str(f))
    assert rc == 0, err
    rc, out_n, err = cli("count", "--kernel", "numba", "--width", "8", str(f))
    assert rc == 0 and out_b == out_n, (out_b, out_n, err)
    rc, out, err = cli("kernels")
    assert rc == 0 and "b200" in out, out + err
    rc, out, err = cli("bench", "--kernels", "b200,numba,baseline", "--sizes", "4k,1m",
                       "--min-time", "0.05")
    assert rc == 0, err
    rows = [ln for ln in out.splitlines() if ln.startswith("b200,")]
    assert len(rows) == 2, out


def test_reference_bench_harness_gpu_columns(ref):
    """bench._resolve_runner("b200") + bench_one (bench.py:113-160) time the
    b200 kernel through the reference harness; ref_plugin.write_csv_gpu adds
    the GPU columns (gpus, hbm_frac, words_per_sec) to the reference's CSV
    schema (bench.py:28-29)."""
    P, k = ref
    from pospopcnt import bench as rb

    from paper_2412_16370_b200 import ref_plugin
    assert rb._resolve_runner("b200") == k.run
    res = [rb.bench_one("b200", s, 16, 0.05, random_fill=True, seed=3) for s in (4096, 1 << 24)]
    res.append(rb.bench_one("numba", 1 << 24, 16, 0.05))
    buf = io.StringIO()
    ref_plugin.write_csv_gpu(res, buf, peak_gbs=6546.2)
    lines = buf.getvalue().splitlines()
    assert lines[0] == ",".join(rb.CSV_COLUMNS + ref_plugin.GPU_COLUMNS)
    cells = [ln.split(",") for ln in lines[1:]]
    assert [c[0] for c in cells] == ["b200", "b200", "numba"]
    assert cells[0][len(rb.CSV_COLUMNS)] == "1" and cells[2][len(rb.CSV_COLUMNS)] == "0"
    for c, r in zip(cells, res):
        wps = float(c[-1])
        assert abs(wps - r.bytes_per_sec / 2) < 1e-6 * wps
    assert cells[2][len(rb.CSV_COLUMNS) + 1] == ""  # no HBM fraction for a CPU kernel
