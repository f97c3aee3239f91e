"""Host-side API contract (no GPU needed): names, validation and error classes
mirror the reference (pkg/tests/test_core.py, test_kernels.py:153-215), and the
product fails loudly instead of falling back to the CPU."""

import os

import numpy as np
import pytest

import paper_2412_16370_b200 as pp
from paper_2412_16370_b200 import core, kernels
from paper_2412_16370_b200.core import InputView

REF_API = ["InputLengthError", "InputView", "KERNEL_ENV", "KernelUnavailableError",
           "UnknownKernelError", "WORD_WIDTHS", "get_kernel", "list_kernels", "new_counters",
           "pospopcnt", "scalar_pospopcnt", "select_kernel", "total_popcount_of",
           "__version__"]


def test_reference_public_names_present():
    """Every name of the reference's __all__ (pospopcnt/__init__.py:22-37)."""
    for name in REF_API:
        assert hasattr(pp, name), name
    assert pp.WORD_WIDTHS == (8, 16, 32, 64)
    assert pp.KERNEL_ENV == "POSPOPCNT_KERNEL"
    assert issubclass(pp.InputLengthError, ValueError)
    assert issubclass(pp.UnknownKernelError, ValueError)
    assert issubclass(pp.KernelUnavailableError, RuntimeError)


def test_scalar_examples():
    """pkg/tests/test_core.py:14-20 known answers on the API's scalar_pospopcnt."""
    assert pp.scalar_pospopcnt(b"\x01\x80", 16) == [1] + [0] * 14 + [1]
    assert pp.scalar_pospopcnt(b"\xff\xff", 16) == [1] * 16
    assert pp.scalar_pospopcnt(b"", 8) == [0] * 8
    c = [3] * 8
    assert pp.scalar_pospopcnt(b"\x0f", 8, c) is c
    assert c == [4, 4, 4, 4, 3, 3, 3, 3]
    assert pp.total_popcount_of([1, 2, 3]) == 6
    assert pp.new_counters(32) == [0] * 32
    with pytest.raises(ValueError):
        pp.new_counters(12)


def test_width_refinement_and_additivity():
    """test_core.py:66-72: C_w[j] = C_2w[j] + C_2w[j+w]; splits add up."""
    rng = np.random.default_rng(1)
    data = rng.integers(0, 256, 4096, dtype=np.uint8).tobytes()
    for w in (8, 16, 32):
        a = pp.scalar_pospopcnt(data, w)
        b = pp.scalar_pospopcnt(data, 2 * w)
        assert a == [b[j] + b[j + w] for j in range(w)]
    c = pp.scalar_pospopcnt(data[:1000], 8)
    pp.scalar_pospopcnt(data[1000:], 8, c)
    assert c == pp.scalar_pospopcnt(data, 8)


def test_inputview_validation():
    base = bytes(100)
    v = InputView(base, 10, 20)
    assert bytes(v.mv()) == bytes(20)
    with pytest.raises(ValueError):
        InputView(base, -1, 5)
    with pytest.raises(ValueError):
        InputView(base, 90, 20)
    assert InputView.of(v) is v
    assert InputView.of(base).nbytes == 100
    with pytest.raises(pp.InputLengthError):
        InputView(base, 0, 7).check_complete(64)
    InputView(base, 0, 8).check_complete(64)


def test_inputview_nbytes_of_arrays_and_tensors():
    """len() of a non-byte buffer counts elements; the view must count bytes
    (SURVEY.md 8a row a2 pitfall)."""
    import torch
    assert InputView.of(np.zeros(10, dtype=np.uint16)).nbytes == 20
    assert InputView.of(torch.zeros(10, dtype=torch.int16)).nbytes == 20
    assert InputView.of(torch.zeros((3, 4), dtype=torch.uint8)).nbytes == 12
    assert InputView.of(memoryview(np.zeros(4, dtype=np.uint32))).nbytes == 16
    assert not InputView.of(torch.zeros(4, dtype=torch.uint8)).on_device


def test_foreign_view_is_adopted():
    """The reference passes its own InputView to kernel.run (kernels.py:333)."""
    from dataclasses import dataclass

    @dataclass(frozen=True)
    class RefView:  # shape of pospopcnt.core.InputView
        base: object
        offset: int
        nbytes: int

    v = InputView.of(RefView(b"abcdefgh", 2, 4))
    assert isinstance(v, InputView) and bytes(v.mv()) == b"cdef"


def test_reference_package_drives_b200_kernel_object():
    """Load the unmodified reference (build container only) and hand it our
    kernel object: validation, dispatch and error classes are the reference's."""
    import importlib.util
    import sys
    src = "/root/reference/pkg/src/pospopcnt"
    if not os.path.exists(src):
        pytest.skip("reference not mounted here")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/pospopcnt_ref_numba_cache")
    spec = importlib.util.spec_from_file_location(
        "pospopcnt_ref_t", os.path.join(src, "__init__.py"), submodule_search_locations=[src])
    ref = importlib.util.module_from_spec(spec)
    sys.modules["pospopcnt_ref_t"] = ref
    old = sys.dont_write_bytecode
    sys.dont_write_bytecode = True  # never write into the reference tree
    try:
        spec.loader.exec_module(ref)
        _drive_reference(ref)
    finally:
        sys.dont_write_bytecode = old


def _drive_reference(ref):
    k = kernels.B200Kernel()
    with pytest.raises(ref.InputLengthError):
        ref.pospopcnt(b"\x00" * 7, 64, kernel=k)
    if not k.available():
        with pytest.raises(ref.KernelUnavailableError):
            ref.pospopcnt(b"\x01\x80", 16, kernel=k)
    # register into the reference's own registry
    from paper_2412_16370_b200.ref_plugin import register
    reg_k = register(ref)
    assert register(ref) is reg_k  # idempotent
    assert ref.get_kernel("b200") is reg_k
    names = [d.name for d, _ in ref.list_kernels()]
    assert names[0] == "portable" and "b200" in names  # reference contract kept
    assert ref.select_kernel().name != "b200"  # default dispatch unchanged
    from importlib import import_module
    ref_bench = import_module("pospopcnt_ref_t.bench")
    if reg_k.available():
        assert callable(ref_bench._resolve_runner("b200"))
    else:
        with pytest.raises(ref.KernelUnavailableError):
            ref_bench._resolve_runner("b200")
        with pytest.raises(ref.KernelUnavailableError):
            ref.select_kernel("b200")


def test_registry_contract(monkeypatch):
    """kernels.py:276-312 semantics with the one B200 kernel."""
    pairs = pp.list_kernels()
    assert [d.name for d, _ in pairs] == ["b200"]
    for d, _ in pairs:
        assert d.block_bytes == 2 * d.r and d.r >= 64
    assert pp.get_kernel("b200").name == "b200"
    with pytest.raises(pp.UnknownKernelError):
        pp.get_kernel("numba")
    with pytest.raises(pp.UnknownKernelError):
        pp.select_kernel("no-such")
    monkeypatch.setenv(pp.KERNEL_ENV, "bogus")
    with pytest.raises(pp.UnknownKernelError):
        pp.select_kernel()


def _gpu_present():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


@pytest.mark.skipif(_gpu_present(), reason="checks the no-GPU behaviour")
def test_no_gpu_means_loud_failure_not_fallback(monkeypatch):
    """Without an sm_100 device there is no CPU fallback: pospopcnt raises."""
    monkeypatch.delenv(pp.KERNEL_ENV, raising=False)
    k = pp.get_kernel("b200")
    assert k.available() is False
    with pytest.raises(pp.KernelUnavailableError):
        pp.pospopcnt(b"\x01\x80", 16)
    with pytest.raises(pp.KernelUnavailableError):
        pp.select_kernel("b200")
    with pytest.raises(pp.KernelUnavailableError):
        pp.pospopcnt(b"\x01\x80", 16, kernel=k)


def test_validation_happens_before_the_kernel():
    """Same error classes and order as kernels.py:315-333, with or without a GPU."""
    with pytest.raises(pp.InputLengthError):
        pp.pospopcnt(b"\x00" * 7, 64)
    with pytest.raises(ValueError):
        pp.pospopcnt(b"\x00" * 8, 12)
    with pytest.raises(ValueError):
        pp.pospopcnt(b"\x00" * 16, 16, counters=[0] * 8)

    class Dead(kernels.B200Kernel):
        def available(self):
            return False

    with pytest.raises(pp.KernelUnavailableError):
        pp.pospopcnt(b"\x00" * 8, 8, kernel=Dead())


def test_b200_kernel_rejects_instrumentation():
    """Like the numba kernel (kernels.py:243-244 / test_kernels.py:180-185)."""
    k = pp.get_kernel("b200")
    with pytest.raises(ValueError):
        k.run(InputView.of(b"\x00" * 16), 8, [0] * 8, fa=lambda a, b, c: (a, b))
    with pytest.raises(ValueError):
        k.run(InputView.of(b"\x00" * 16), 8, [0] * 8, probe=print)


def test_reference_protocol_shape():
    """The kernel object satisfies the reference's duck-typed protocol
    (name, r, descriptor, available(), run(view, w, counters))."""
    k = kernels.B200Kernel()
    assert isinstance(k.name, str) and isinstance(k.r, int)
    assert callable(k.available) and callable(k.run)
    assert k.descriptor.name == "b200"
    assert repr(k) == "<kernel b200 r=128>"


def test_package_never_imports_oracle():
    """The oracle is test infrastructure; the product must not touch it."""
    import re
    pkg = os.path.dirname(pp.__file__)
    bad = re.compile(r"(from\s+oracle|import\s+oracle|liboracle|oracle_\w+\s*\(|"
                     r"pospopcnt_oracle\.h)")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(root, f)).read()
                assert not bad.search(src), f


def test_shard_ranges_cover_and_align():
    from paper_2412_16370_b200.dist import shard_range
    for total in (0, 64, 1000, 1 << 20, (1 << 30) + 8):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, _) in zip(spans, spans[1:]):
                assert b == c and a <= b and b % 64 == 0
    with pytest.raises(ValueError):
        shard_range(100, 2, 2)


@pytest.mark.skipif(_gpu_present(), reason="checks the no-GPU behaviour")
def test_categories_and_segments_fail_loudly_without_gpu():
    import numpy as np
    with pytest.raises(pp.KernelUnavailableError):
        pp.pospopcnt_categories(np.zeros(16, dtype=np.uint8), 8)
    with pytest.raises(ValueError):
        pp.pospopcnt_categories(np.zeros(16, dtype=np.uint8), 12)
    with pytest.raises(ValueError):  # segmented counting needs device data
        pp.pospopcnt_segmented(b"\x00" * 16, [0, 8, 16], 8)


def test_segmented_launch_shape_rule():
    """Host-side shape rule of the segmented entry points: one lane per array
    when every array is tiny, else G by the byte-weighted mean length
    (profiles/r1_segmented_ablation.md)."""
    import numpy as np
    from paper_2412_16370_b200 import segmented as S
    rng = np.random.default_rng(3)
    K = 1024

    def g(lens, aligned=False):
        lens = np.asarray(lens, dtype=np.int64)
        return S._shape(lens.size, int(lens.max()), S._byte_mean(lens), aligned)[0]

    assert g(np.full(1000, 64)) == 1
    assert g(np.full(1000, 4 * K)) == 8
    assert g(np.full(1000, 8 * K)) == 16
    assert g(np.full(1000, 16 * K)) == 32
    assert g(rng.integers(0, 16 * K // 8, 100_000) * 8) == 32   # byte mean 10.7 KiB
    assert g(rng.integers(4 * K // 8, 12 * K // 8, 100_000) * 8) == 16
    assert g(rng.integers(0, 8 * K // 8, 100_000) * 8) == 8     # byte mean 5.3 KiB
    assert S._byte_mean(np.array([0, 0])) == 0.0
    assert S._byte_mean(np.array([2, 6])) == 5.0


def test_segmented_hybrid_rule():
    """Mostly-tiny arrays take the hybrid split with G = 32 for the rest."""
    import numpy as np
    from paper_2412_16370_b200 import segmented as S
    rng = np.random.default_rng(4)

    def shape(lens):
        lens = np.asarray(lens, dtype=np.int64)
        return S._shape(lens.size, int(lens.max()), S._byte_mean(lens), False,
                        int(np.count_nonzero(lens <= S.LANE_MAX_BYTES)))

    assert shape(np.where(rng.random(10_000) < 0.9, 64, 16384)) == (32, True)
    assert shape(np.where(rng.random(10_000) < 0.7, 256, 4096)) == (32, True)
    assert shape(np.where(rng.random(10_000) < 0.5, 512, 2048)) == (8, False)
    assert shape(np.full(100, 256)) == (1, False)


def test_segment_plan_order():
    """SegmentPlan's processing order: a permutation; each full group of
    32/G slots holds segments adjacent in length-sorted order; long and short
    groups alternate; the partial group goes last."""
    import numpy as np
    from paper_2412_16370_b200.segmented import SegmentPlan
    rng = np.random.default_rng(9)
    d = rng.integers(0, 5000, 1003)
    for S in (1, 2, 4):
        order = SegmentPlan._order(d, S)
        assert sorted(order.tolist()) == list(range(d.size))
        rank = np.empty(d.size, dtype=np.int64)
        rank[np.argsort(-d, kind="stable")] = np.arange(d.size)
        nfull = d.size // S
        groups = rank[order[: nfull * S]].reshape(nfull, S)
        assert (groups.max(1) - groups.min(1) == S - 1).all()  # neighbours in sorted order
        first = groups.min(1) // S  # the sorted group each slot group came from
        assert first[0] == 0 and (nfull < 2 or first[1] == nfull - 1)
        assert sorted(first.tolist()) == list(range(nfull))
        assert set(rank[order[nfull * S:]].tolist()) == set(range(nfull * S, d.size))


def test_segment_plan_shape():
    """SegmentPlan's shape rule (built on the CPU: no launch needed)."""
    import numpy as np
    from paper_2412_16370_b200.segmented import SegmentPlan
    rng = np.random.default_rng(10)
    K = 1024

    def plan(lens):
        offs = np.zeros(len(lens) + 1, dtype=np.int64)
        offs[1:] = np.cumsum(lens)
        return SegmentPlan(offs, device="cpu")

    assert plan(rng.integers(0, 16 * K // 8, 20_000) * 8).lanes == 8    # byte mean 10.7 K
    assert plan(rng.integers(0, 32 * K // 8, 20_000) * 8).lanes == 16   # 21 K
    assert plan(np.full(1000, 64 * K)).lanes == 32
    p = plan(np.where(rng.random(20_000) < 0.9, 64, 16 * K))
    assert (p.lanes, p.hybrid) == (32, True)
    assert plan(np.full(1000, 256)).lanes == 1
    assert plan(np.full(10, 4096)).order.numel() == 10


def test_devices_argument_parsing(monkeypatch):
    """pospopcnt(..., devices=) / B200Kernel(devices=) / POSPOPCNT_B200_DEVICES:
    host inputs fanned out over several GPUs (pp_count_host_multi)."""
    from paper_2412_16370_b200 import kernels as K
    monkeypatch.delenv(K.DEVICES_ENV, raising=False)
    assert K._resolve_devices(None) is None
    assert K._resolve_devices([0, 0, 1]) == (0, 0, 1)
    assert K._resolve_devices("1, 2") == (1, 2)
    monkeypatch.setenv(K.DEVICES_ENV, "0,3")
    assert K._resolve_devices(None) == (0, 3)
    with pytest.raises(ValueError):
        K._resolve_devices([])
    with pytest.raises(ValueError):
        K._resolve_devices([0] * 17)
    with pytest.raises(ValueError):  # another kernel cannot take devices=
        K.pospopcnt(b"\x00" * 8, 8, kernel=object(), devices=[0])
