"""CPU legs of bench.py: the reference's own CPU implementation, timed on the
box's host cores.

Two implementations of the same CPU path:

* ``kind: "reference"`` -- the UNMODIFIED reference package (pospopcnt 0.1.0,
  /root/reference/pkg) installed into ``baseline/_ref`` (git-ignored; it
  travels to the GPU box with the snapshot), called through its own public
  API ``pospopcnt.pospopcnt(InputView(...), w, kernel=...)``
  (pkg/src/pospopcnt/kernels.py:315-333).  Its fastest kernel is numba
  (kernels.py:218-270, _nbkern.py:43-177); it holds the GIL, so the P-core
  row forks P processes over contiguous 64-byte-cut shards of one shared
  buffer (additivity), the numba code compiled once in the parent
  before the fork.
* ``kind: "port"`` -- the C restatement of the same algorithm under
  ``oracle/`` (test infrastructure), on P threads: used only when
  ``baseline/_ref`` (or numba) is missing.

Rows: ``ref-numba-Pcore`` (the reported value),
``ref-numba-1core``, ``ref-default`` (default dispatch = the numpy kernel,
kernels.py:300-312 -> 178-215) and ``ref-scalar`` (core.py:82-96, C1 only).
Methodology of the reference harness (bench.py:124-160): k doubles until a
round lasts >= min_time, >= 2 rounds, the last one reported; the first-call
JIT is excluded.
"""

import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    import platform
    return platform.processor() or "unknown"


def host_info():
    return {"cpu_model": cpu_model(), "threads_usable": host_threads(),
            "cpu_count": os.cpu_count()}


_REF = None


def load_reference():
    """(module, None) for the installed reference with a working numba
    kernel, or (None, why)."""
    global _REF
    if _REF is not None:
        return _REF
    if not os.path.isdir(os.path.join(REF_DIR, "pospopcnt")):
        _REF = (None, "baseline/_ref not installed (scripts/stage_reference.sh)")
        return _REF
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/pp_numba_cache")
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import importlib
        ref = importlib.import_module("pospopcnt")
        if not os.path.abspath(ref.__file__).startswith(REF_DIR):
            raise ImportError(f"imported {ref.__file__}, not baseline/_ref")
        if not ref.get_kernel("numba").available():
            raise ImportError("numba kernel unavailable")
        # first-call JIT (excluded from every timing, as in the reference harness)
        ref.pospopcnt(bytes(range(256)) * 64, 8, kernel="numba")
        _REF = (ref, None)
    except Exception as exc:  # noqa: BLE001
        _REF = (None, f"reference import failed: {exc}")
    return _REF


def _geometric(one, min_time):
    """k doubles until a round lasts >= min_time; >= 2 rounds; last reported."""
    k, rounds = 1, 0
    while True:
        t0 = time.perf_counter()
        for _ in range(k):
            one()
        t = time.perf_counter() - t0
        rounds += 1
        if rounds >= 2 and t >= min_time:
            return k, t
        k = k * 2 if 2 * t < min_time else max(k + 1, int(k * min_time / max(t, 1e-9) * 1.05) + 1)


def _cuts(nbytes, parts, align=64):
    units = nbytes // align
    return [(units * i // parts * align, nbytes if i == parts - 1 else units * (i + 1) // parts * align)
            for i in range(parts)]


# ---- P-process numba reference over one shared buffer (fork) --------------
_SHARED = {}


def _child(i, lo, hi, w, seg, steps, warmup, start, end, q):
    ref = _REF[0]
    host = _SHARED["host"]
    try:
        def one():
            if seg:
                for s in range(lo, hi, seg):
                    ref.pospopcnt(ref.InputView(host, s, seg), w, kernel="numba")
                return None
            return ref.pospopcnt(ref.InputView(host, lo, hi - lo), w, kernel="numba")
        for _ in range(warmup):
            one()
        res = one()
        start.wait()
        for _ in range(steps):
            one()
        end.wait()
        q.put((i, res))
    except Exception as exc:  # noqa: BLE001
        q.put((i, exc))
        start.abort()
        end.abort()


def run_ref_pcore(host, w, steps, warmup, procs=None, seg=0):
    """The reference numba kernel on `procs` forked processes over contiguous
    shards of `host` (u8 numpy array).  Returns (seconds for `steps` passes
    over the whole buffer, summed counters of one pass or None, procs)."""
    ref, why = load_reference()
    if ref is None:
        raise RuntimeError(why)
    procs = procs or host_threads()
    align = max(64, seg) if seg else 64
    cuts = _cuts(host.size, procs, align)
    cuts = [c for c in cuts if c[1] > c[0]]
    ctx = mp.get_context("fork")
    start, end = ctx.Barrier(len(cuts) + 1), ctx.Barrier(len(cuts) + 1)
    q = ctx.Queue()
    _SHARED["host"] = host
    ps = [ctx.Process(target=_child, args=(i, lo, hi, w, seg, steps, warmup, start, end, q),
                      daemon=True) for i, (lo, hi) in enumerate(cuts)]
    for p in ps:
        p.start()
    try:
        start.wait(timeout=600)
        t0 = time.perf_counter()
        end.wait(timeout=3600)
        t = time.perf_counter() - t0
    except Exception as exc:  # noqa: BLE001
        for p in ps:
            p.kill()
        raise RuntimeError(f"reference worker failed: {exc}") from exc
    res = [q.get(timeout=60) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    _SHARED.clear()
    total = None
    for _, r in sorted(res, key=lambda x: x[0]):
        if isinstance(r, Exception):
            raise r
        if r is not None:
            total = list(r) if total is None else [a + b for a, b in zip(total, r)]
    return t, total, len(cuts)


def ref_rows(host, w, min_time=2.0, scalar=False):
    """The single-process rows of BASELINE.md section 3 on `host` (a bounded
    sample): numba on one core, default dispatch (numpy kernel), and the
    scalar restatement when asked (C1).  Returns {row: {...}}."""
    ref, why = load_reference()
    if ref is None:
        return {"unavailable": why}
    rows = {}
    view = ref.InputView(host, 0, host.size)
    k, t = _geometric(lambda: ref.pospopcnt(view, w, kernel="numba"), min_time)
    rows["ref-numba-1core"] = {"GBs": round(host.size * k / t / 1e9, 3), "cores": 1,
                               "sample": f"{host.size >> 20} MiB x {k} in {t:.2f} s"}
    default = ref.select_kernel(None)
    n_np = min(host.size, 64 << 20)
    vnp = ref.InputView(host, 0, n_np)
    k, t = _geometric(lambda: ref.pospopcnt(vnp, w), min_time)
    rows["ref-default"] = {"GBs": round(n_np * k / t / 1e9, 3), "cores": 1,
                           "kernel": default.name,
                           "sample": f"{n_np >> 20} MiB x {k} in {t:.2f} s"}
    if scalar:
        n_sc = min(host.size, 256 << 10)
        mv = memoryview(host[:n_sc])
        k, t = _geometric(lambda: ref.scalar_pospopcnt(mv, w), min_time / 4)
        rows["ref-scalar"] = {"GBs": round(n_sc * k / t / 1e9, 6), "cores": 1,
                              "sample": f"{n_sc >> 10} KiB x {k} in {t:.2f} s"}
    return rows


def port_pcore(host, w, min_time, seg=0):
    """Fallback: the C port under oracle/ on all host threads (kind "port")."""
    import numpy as np
    from oracle import oracle as O
    threads = host_threads()
    if seg:
        offs = np.arange(host.size // seg + 1, dtype=np.uint64) * seg
        one = lambda: O.segments(host, offs, w, threads=threads)  # noqa: E731
    else:
        one = lambda: O.hs512(host, 0, host.size, w, threads=threads)  # noqa: E731
    once = one()
    k, t = _geometric(one, min_time)
    return host.size * k / t / 1e9, threads, once, k, t
