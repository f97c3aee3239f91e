"""Register the B200 kernel inside the reference package.

The reference resolves kernels by name only from its module-level registry
(kernels.py:276-285, ``_KERNELS`` filled by ``_registry()``), which drives
``get_kernel``/``select_kernel``/``POSPOPCNT_KERNEL`` (kernels.py:288-312),
its benchmark harness (``bench._resolve_runner``, bench.py:113-121) and its
selftest (selftest.py:44-90).  ``register(ref)`` appends a ``B200Kernel`` to
that registry without editing the reference's files, so

    pospopcnt bench --kernels b200,numba,baseline
    POSPOPCNT_KERNEL=b200 pospopcnt count FILE

run the sm_100a kernel unchanged.  (The reference's default dispatch picks
the kernel with the widest ``r``; the B200 kernel reports r=128 and so never
displaces the reference's own default unless selected by name.)
"""

from .kernels import B200Kernel

# columns appended to the reference's benchmark CSV (bench.py:28-29) for the
# GPU rows: GPUs used by the row's kernel, its input rate as a fraction of
# the HBM peak (empty for CPU kernels), and words/s at the row's width
GPU_COLUMNS = ("gpus", "hbm_frac", "words_per_sec")


def register(ref):
    """Add the B200 kernel to the reference module ``ref`` (idempotent).

    ``ref`` is the imported reference package (``import pospopcnt``) or its
    ``kernels`` submodule.  Returns the registered kernel object.
    """
    km = getattr(ref, "kernels", ref)
    reg = km._registry()  # materialise the built-in list first (kernels.py:276)
    for k in reg:
        if getattr(k, "name", None) == B200Kernel.name:
            return k
    k = B200Kernel()
    reg.append(k)
    return k


def gpu_cells(result, peak_gbs, gpus=None):
    """The GPU_COLUMNS cells of one reference BenchResult (bench.py:83-110)."""
    on_gpu = result.kernel == B200Kernel.name
    n = (gpus if gpus is not None else 1) if on_gpu else 0
    frac = "" if not on_gpu or not peak_gbs else repr(result.bytes_per_sec / 1e9 / peak_gbs)
    return [str(n), frac, repr(result.bytes_per_sec / (result.width // 8))]


def write_csv_gpu(results, out, peak_gbs=None, hw=None, gpus=None):
    """The reference's CSV (bench.write_csv, bench.py:213-219) with
    GPU_COLUMNS appended to the header and to every row.  ``peak_gbs``: the
    HBM roofline (e.g. MEASURED_PEAKS.json hbm_gbs); ``gpus``: devices the
    b200 rows used (default 1)."""
    import importlib
    rb = importlib.import_module(type(results[0]).__module__) if results else None
    if hw is None:
        hw = any(getattr(r, "cycles", None) is not None for r in results)
    header = rb.csv_header(hw) if rb is not None else ""
    out.write(header + "," + ",".join(GPU_COLUMNS) + "\n")
    for r in results:
        out.write(r.csv_row(hw) + "," + ",".join(gpu_cells(r, peak_gbs, gpus)) + "\n")
