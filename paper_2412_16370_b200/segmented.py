"""Segmented (many-small-arrays) counting: one launch, one counter row per array.

New relative to the reference, which counts one array per call
(kernels.py:315-333) and takes its short-array path for anything below 15
vectors (edges.py:96-102, kernels.py:249-250).  Calling the reference once
per segment and collecting each counter list is the semantics reproduced
here: row s of the output equals ``pospopcnt(segment_s, width)``.

Segments live in one CUDA byte buffer; segment s is bytes
[offsets[s], offsets[s+1]) of the view.  Every segment must be word-complete.
"""

import collections
import hashlib
import threading
import weakref

import numpy as np

from . import _lib
from .core import InputLengthError, InputView, check_width, is_torch_tensor

# arrays up to this many bytes are counted one lane each (pp_seglane_kernel);
# when every array starts and ends on a 16-byte boundary the G-lane kernels
# win above LANE_MAX_ALIGNED (no partial vectors).  The C ABI applies the same
# bounds to fixed-size segments (scripts/seg_smallG.py).
LANE_MAX_BYTES = 512
LANE_MAX_ALIGNED = 512


def _device_view(data):
    view = InputView.of(data)
    if not view.on_device:
        raise ValueError("segmented counting needs the data in a CUDA tensor "
                         "(copy it once with torch.as_tensor(...).cuda())")
    if not view.base.is_contiguous():
        raise ValueError("input tensor must be contiguous")
    return view


def _out_tensor(out, nseg, width, device):
    import torch
    if out is None:
        return torch.zeros((nseg, width), dtype=torch.int64, device=device), True
    if not (is_torch_tensor(out) and out.is_cuda and out.device == device):
        raise ValueError("out must be a CUDA tensor on the data's device")
    if out.dtype not in (torch.int64, torch.uint64) or not out.is_contiguous():
        raise ValueError("out must be a contiguous int64/uint64 tensor")
    if out.numel() < nseg * width:
        raise ValueError(f"out holds {out.numel()} < {nseg * width} counters")
    return out, False


def pospopcnt_segmented(data, offsets, width, out=None, accumulate=True, validate=True,
                        lanes=None, hybrid=None, plan=None):
    """Positional counts of many arrays in one launch.

    ``offsets``: nseg+1 non-decreasing byte offsets into the view (host
    sequence / numpy array, or a CUDA int64 tensor).  ``out``: CUDA
    (nseg, width) int64 tensor accumulated into (or overwritten when
    ``accumulate=False``); allocated zeroed when None.  Returns ``out``.
    Asynchronous on the current stream.  ``lanes`` (1, 8, 16 or 32) forces
    the lanes-per-segment launch shape.  By default it follows the segment
    lengths (host offsets, or device offsets with ``validate``): one lane per
    segment when every segment is at most LANE_MAX_BYTES, else G lanes by the
    byte-weighted mean length (_shape); unknown lengths (device offsets, ``validate=False``) get the
    C ABI default, G = 8.  ``hybrid=True`` adds a one-lane pass for the
    segments of at most LANE_MAX_BYTES (PP_SEG_HYBRID), which pays when
    most arrays are that small; ``None`` (default) lets the shape rule
    decide when the lengths are known (``_shape``), ``False`` never.
    ``plan``: a ``SegmentPlan`` built once for these offsets (repeated counts
    over one segmentation): the G-lane kernel then takes the segments in the
    plan's length-sorted order and the plan's shape; ``offsets`` may be None.
    Default (``plan=None``): a ragged segmentation counted a second time
    with the same offsets (the same, unmodified CUDA tensor, or equal host
    offsets) and the default shape gets a ``SegmentPlan`` built and cached
    (``PLAN_CACHE_SIZE`` most recent segmentations per process) and used
    from then on; ``plan=False`` never plans.
    """
    import torch
    check_width(width)
    view = _device_view(data)
    if plan is not None and plan is not False:
        return plan.count(view, width, out=out, accumulate=accumulate)
    auto = plan is None and lanes is None and hybrid is None
    if auto:
        cached = _PLANS.lookup(offsets, view.base.device)
        if cached is not None:
            return cached.count(view, width, out=out, accumulate=accumulate)
    dev = view.base.device
    step = width // 8
    shape = None  # (lanes, hybrid) from the lengths, when they are known here
    if is_torch_tensor(offsets) and offsets.is_cuda:
        offs = offsets.to(torch.int64).contiguous()
        if validate and offs.numel() > 1:
            d = offs[1:] - offs[:-1]
            bad_order = bool((d < 0).any()) or int(offs[0]) < 0 or int(offs[-1]) > view.nbytes
            if bad_order:
                raise ValueError("offsets must be non-decreasing and inside the view")
            if bool(((d & (step - 1)) != 0).any()):
                raise InputLengthError(f"a segment is not a multiple of the {step}-byte word size")
            if lanes is None:  # validation already synchronised: pick the shape too
                shape = _shape(int(d.numel()), int(d.max()), _byte_mean(d),
                               _aligned_offsets(view, offs),
                               int((d <= LANE_MAX_BYTES).sum()))
    else:
        offs_np = np.asarray(offsets, dtype=np.int64)
        if offs_np.ndim != 1 or offs_np.size < 1:
            raise ValueError("offsets must be a 1-D sequence of nseg+1 byte offsets")
        d = np.diff(offs_np) if (validate or lanes is None) else None
        if validate:
            if (d < 0).any() or offs_np[0] < 0 or offs_np[-1] > view.nbytes:
                raise ValueError("offsets must be non-decreasing and inside the view")
            if (d & (step - 1)).any():
                raise InputLengthError(f"a segment is not a multiple of the {step}-byte word size")
        offs = torch.as_tensor(offs_np, device=dev)
        if lanes is None and offs_np.size > 1:
            shape = _shape(int(d.size), int(d.max()), _byte_mean(d),
                           _aligned_offsets(view, offs_np),
                           int(np.count_nonzero(d <= LANE_MAX_BYTES)))
    nseg = offs.numel() - 1
    out, fresh = _out_tensor(out, max(nseg, 0), width, dev)
    if nseg <= 0:
        return out
    lib = _lib.load()
    flags = _lib.PP_SEG_ACCUMULATE if (accumulate and not fresh) else _lib.PP_SEG_OVERWRITE
    if auto and shape is not None and shape[0] != 1 and not shape[1] and nseg >= 64:
        # G-lane shape over ragged lengths: the length-sorted plan pays when
        # the same segmentation comes back (built on the second sighting)
        _PLANS.seen(offsets, dev, d)
    if lanes is None and shape is not None:
        lanes = shape[0]
        if hybrid is None:
            hybrid = shape[1]
    if hybrid:
        flags |= _lib.PP_SEG_HYBRID
    flags |= _lanes_flag(lanes)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        base_ptr = view.base.data_ptr() + view.offset
        _lib.check(lib.pp_count_segmented(base_ptr, offs.data_ptr(), nseg, width,
                                          out.data_ptr(), flags, stream))
        # keep the offsets tensor alive until the kernel has consumed it
        offs.record_stream(torch.cuda.current_stream(dev))
    return out


PLAN_CACHE_SIZE = 8


class _PlanCache:
    """Segmentations seen by pospopcnt_segmented, and the plans built for
    those seen twice.  A CUDA offsets tensor is keyed by identity plus its
    version counter (an in-place write invalidates the entry; a freed
    tensor's entry dies with its weakref); host offsets by their bytes.
    Thread-safe; ``stats`` = [plans built, plan hits]."""

    def __init__(self, size):
        self.size = size
        self.lock = threading.Lock()
        self.seen_keys = collections.OrderedDict()  # key -> None (first sighting)
        self.plans = collections.OrderedDict()      # key -> (check, SegmentPlan)
        self.stats = [0, 0]

    @staticmethod
    def _key(offsets, dev):
        if is_torch_tensor(offsets):
            if not offsets.is_cuda:
                offsets = offsets.numpy()
            else:
                return (("dev", id(offsets), offsets._version, str(dev)),
                        weakref.ref(offsets))
        a = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
        return ("host", a.size, hashlib.blake2b(a.data, digest_size=16).digest(), str(dev)), None

    def lookup(self, offsets, dev):
        key, ref = self._key(offsets, dev)
        with self.lock:
            hit = self.plans.get(key)
            if hit is None:
                return None
            if hit[0] is not None and hit[0]() is not offsets:  # id reused by a new tensor
                del self.plans[key]
                return None
            self.plans.move_to_end(key)
            self.stats[1] += 1
            return hit[1]

    def seen(self, offsets, dev, lengths):
        key, ref = self._key(offsets, dev)
        with self.lock:
            if key not in self.seen_keys:
                self.seen_keys[key] = ref
                while len(self.seen_keys) > 4 * self.size:
                    self.seen_keys.popitem(last=False)
                return
            first = self.seen_keys.pop(key)
            if first is not None and first() is not offsets:
                self.seen_keys[key] = ref
                return
        if is_torch_tensor(lengths):
            lengths = lengths.cpu().numpy()
        if int(lengths.min()) == int(lengths.max()):
            return  # equal lengths: index order is already balanced
        p = SegmentPlan(offsets, device=dev)
        with self.lock:
            self.plans[key] = (ref, p)
            self.stats[0] += 1
            while len(self.plans) > self.size:
                self.plans.popitem(last=False)

    def clear(self):
        with self.lock:
            self.seen_keys.clear()
            self.plans.clear()
            self.stats = [0, 0]


_PLANS = _PlanCache(PLAN_CACHE_SIZE)


def _byte_mean(d):
    """Byte-weighted mean length sum(L^2) / sum(L): the length of the array
    an average byte belongs to (numpy array or CUDA tensor of lengths)."""
    if is_torch_tensor(d):
        tot = int(d.sum())
        return float((d.double() ** 2).sum()) / tot if tot else 0.0
    d = np.asarray(d, dtype=np.float64)
    tot = d.sum()
    return float((d * d).sum() / tot) if tot else 0.0


def _shape(nseg, dmax, bmean, vec_aligned, nshort=0):
    """Launch shape from the length distribution: (lanes, hybrid).

    Every array <= LANE_MAX_BYTES (LANE_MAX_ALIGNED when all arrays are
    16-byte aligned): one lane each, else G lanes by the byte-weighted mean
    length ``bmean`` (sum L^2 / sum L): G = 8 below 6 KiB, 16 below 10 KiB,
    else 32 -- the best G over 11 length distributions, fixed, uniform,
    exponential and log-normal (scripts/seg_shape_sweep.py,
    profiles/r1_segmented_ablation.md); the count mean under-weights the
    long arrays that carry most of the bytes.  When at least 60 % of the
    arrays (``nshort`` of ``nseg``) are at most LANE_MAX_BYTES: the hybrid
    split (PP_SEG_HYBRID: those one lane each in a separate pass) with
    G = 32 for the rest, which skips whole short groups (measured best on
    every such mix, 1.1-1.7x faster: scripts/seg_hybrid_sweep.py); at 50 %
    the split no longer pays.
    """
    if dmax <= (LANE_MAX_ALIGNED if vec_aligned else LANE_MAX_BYTES):
        return 1, False
    if nseg and nshort >= 0.6 * nseg:
        return 32, True
    return (32 if bmean >= 10240 else 16 if bmean >= 6144 else 8), False


def _aligned_offsets(view, offs):
    """Do all segments start on 16-byte boundaries?  Only computed when the
    shape rule depends on it (LANE_MAX_ALIGNED != LANE_MAX_BYTES)."""
    if LANE_MAX_ALIGNED == LANE_MAX_BYTES:
        return False
    if (view.base.data_ptr() + view.offset) % 16:
        return False
    return not bool(((offs & 15) != 0).any())


def _lanes_flag(lanes):
    if lanes is None:
        return 0
    if lanes not in (1, 2, 4, 8, 16, 32):
        raise ValueError("lanes must be 1, 2, 4, 8, 16 or 32")
    return lanes << 8


class SegmentPlan:
    """A reusable launch plan for one CSR segmentation (offsets), for callers
    that count many inputs with the same layout.

    Ragged lengths leave lanes idle: a G-lane group of 32/G segments runs as
    long as its longest member.  The plan sorts the segments by length and
    groups neighbours in that order, so each group's segments have similar
    lengths; groups are then taken long, short, long, short, ... (longest
    first for the tail, and streaming-bound long groups interleaved with
    flush-bound short ones).  ``count`` launches pp_count_segmented_order;
    rows still land at their segment's index.  The shape (lanes, hybrid)
    comes from ``_shape`` (one lane for all-tiny arrays, the hybrid split for
    mostly-tiny ones) with G = 8 / 16 / 32 below 17 / 34 KiB / above of
    byte-weighted mean length, unless ``lanes`` forces it.  Measured vs the
    index order (1 GiB, w=64): uniform 0-4 KiB 373 -> 312 us, exponential
    mean 2 KiB 414 -> 312, mean 4 KiB 294 -> 241 (best G each side).
    """

    def __init__(self, offsets, device=None, lanes=None, hybrid=None):
        import torch
        if is_torch_tensor(offsets):
            device = offsets.device if offsets.is_cuda else device
            offs_np = offsets.detach().cpu().numpy().astype(np.int64)
        else:
            offs_np = np.asarray(offsets, dtype=np.int64)
        if offs_np.ndim != 1 or offs_np.size < 1:
            raise ValueError("offsets must be a 1-D sequence of nseg+1 byte offsets")
        d = np.diff(offs_np)
        if (d < 0).any() or offs_np[0] < 0:
            raise ValueError("offsets must be non-decreasing and non-negative")
        self.nseg = int(d.size)
        if self.nseg >= 1 << 32:
            raise ValueError("a plan holds 32-bit segment indices")
        self.end = int(offs_np[-1])
        # OR of all lengths: word-complete for w iff its low log2(w/8) bits are 0
        self._len_or = int(np.bitwise_or.reduce(d)) if d.size else 0
        if self.nseg:
            bm = _byte_mean(d)
            shp = _shape(self.nseg, int(d.max()), bm, False,
                         int(np.count_nonzero(d <= LANE_MAX_BYTES)))
            if shp[0] != 1 and not shp[1]:
                # balanced groups: 8 lanes per segment stay best to a larger
                # byte mean than in index order (scripts/seg_plan_probe.py)
                shp = (8 if bm < 17 * 1024 else 16 if bm < 34 * 1024 else 32), False
        else:
            shp = (8, False)
        self.lanes = lanes if lanes is not None else shp[0]
        self.hybrid = shp[1] if hybrid is None else bool(hybrid)
        if self.lanes == 1 or self.hybrid:
            # the one-lane kernel takes segments in index order; with the
            # hybrid split the sorted order measured slower (90 % 64 B /
            # 16 KiB: 310 vs 285 us), the G pass skips the tiny groups anyway
            order = np.arange(self.nseg, dtype=np.uint32)
        else:
            order = self._order(d, 32 // self.lanes)
        dev = torch.device(device) if device is not None else torch.device("cuda")
        if dev.type == "cuda" and dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.offsets = torch.as_tensor(offs_np, device=dev)
        self.order = torch.as_tensor(order.view(np.int32), device=dev)

    @staticmethod
    def _order(d, S):
        """Segment indices by descending length, cut into groups of S, the
        full groups taken alternately from the long and the short end, the
        partial group (if any: the S shortest-but-remaining) last."""
        idx = np.argsort(-d, kind="stable").astype(np.uint32)
        nfull = idx.size // S
        full = idx[: nfull * S].reshape(nfull, S)
        g = np.empty(nfull, dtype=np.int64)
        g[0::2] = np.arange((nfull + 1) // 2)
        g[1::2] = nfull - 1 - np.arange(nfull // 2)
        return np.concatenate([full[g].reshape(-1), idx[nfull * S:]])

    def count(self, data, width, out=None, accumulate=True):
        """Positional counts of the plan's segments of ``data`` (as
        pospopcnt_segmented).  Asynchronous on the current stream."""
        import torch
        check_width(width)
        view = _device_view(data)
        if view.base.device != self.device:
            raise ValueError("data and plan live on different devices")
        if self.end > view.nbytes:
            raise ValueError("the plan's offsets run past the view")
        if self._len_or & (width // 8 - 1):
            raise InputLengthError(f"a segment is not a multiple of the {width // 8}-byte "
                                   "word size")
        out, fresh = _out_tensor(out, self.nseg, width, self.device)
        if self.nseg == 0:
            return out
        lib = _lib.load()
        flags = _lib.PP_SEG_ACCUMULATE if (accumulate and not fresh) else _lib.PP_SEG_OVERWRITE
        if self.hybrid:
            flags |= _lib.PP_SEG_HYBRID
        flags |= _lanes_flag(self.lanes)
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device).cuda_stream
            _lib.check(lib.pp_count_segmented_order(
                view.base.data_ptr() + view.offset, self.offsets.data_ptr(),
                self.order.data_ptr(), self.nseg, width, out.data_ptr(), flags, stream))
        return out


def pospopcnt_fixed(data, seg_bytes, width, out=None, accumulate=True, lanes=None):
    """Equal-size segments: segment s = bytes [s*seg_bytes, (s+1)*seg_bytes) of the view.

    A trailing partial segment is not counted (nseg = nbytes // seg_bytes).
    """
    import torch
    check_width(width)
    if seg_bytes <= 0:
        raise ValueError("seg_bytes must be positive")
    if seg_bytes % (width // 8):
        raise InputLengthError(f"{seg_bytes} bytes is not a multiple of the "
                               f"{width // 8}-byte word size")
    view = _device_view(data)
    dev = view.base.device
    nseg = view.nbytes // seg_bytes
    out, fresh = _out_tensor(out, nseg, width, dev)
    if nseg == 0:
        return out
    lib = _lib.load()
    flags = _lib.PP_SEG_ACCUMULATE if (accumulate and not fresh) else _lib.PP_SEG_OVERWRITE
    flags |= _lanes_flag(lanes)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(lib.pp_count_fixed(view.base.data_ptr() + view.offset, seg_bytes, nseg,
                                      width, out.data_ptr(), flags, stream))
    return out


def pospopcnt_batch(arrays, width, out=None, accumulate=True, lanes=None):
    """Positional counts of many separate device arrays in one launch.

    ``arrays``: a sequence of CUDA tensors and/or InputViews over CUDA
    tensors, all on one device, each word-complete.  Row i of the returned
    (n, width) int64 tensor is ``pospopcnt(arrays[i], width)``.  The launch
    shape follows the lengths (one lane per array when all are at most
    LANE_MAX_BYTES, else G lanes by the byte-weighted mean length) unless
    ``lanes`` forces
    it.  Asynchronous on the current stream (the pointer/length table is
    copied to the device once per call).
    """
    import torch
    check_width(width)
    n = len(arrays)
    if n == 0:
        raise ValueError("pospopcnt_batch needs at least one array")
    step = width // 8
    ptrs = np.empty(n, dtype=np.uint64)
    lens = np.empty(n, dtype=np.uint64)
    dev = None
    for i, a in enumerate(arrays):
        if isinstance(a, torch.Tensor):  # fast path: no view object per array
            if not a.is_cuda:
                raise ValueError("pospopcnt_batch needs CUDA tensors")
            if not a.is_contiguous():
                raise ValueError("input tensor must be contiguous")
            d, ptr, nb = a.device, a.data_ptr(), a.numel() * a.element_size()
        else:
            v = _device_view(a)
            d, ptr, nb = v.base.device, v.base.data_ptr() + v.offset, v.nbytes
        if dev is None:
            dev = d
        elif d != dev:
            raise ValueError("all arrays must live on one device")
        ptrs[i] = ptr
        lens[i] = nb
    bad = np.nonzero(lens & np.uint64(step - 1))[0]
    if bad.size:
        i = int(bad[0])
        raise InputLengthError(f"array {i}: {int(lens[i])} bytes is not a multiple of the "
                               f"{step}-byte word size")
    out, fresh = _out_tensor(out, n, width, dev)
    if lanes is None:
        dmax = int(lens.max())
        aligned = not bool(((ptrs % 16) | (lens % 16)).any())
        lanes = _shape(n, dmax, _byte_mean(lens), aligned)[0]
    table = torch.from_numpy(np.concatenate([ptrs, lens]).view(np.int64)).to(dev)
    lib = _lib.load()
    flags = _lib.PP_SEG_ACCUMULATE if (accumulate and not fresh) else _lib.PP_SEG_OVERWRITE
    flags |= _lanes_flag(lanes)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(lib.pp_count_batch(table.data_ptr(), table.data_ptr() + 8 * n, n, width,
                                      out.data_ptr(), flags, stream))
        table.record_stream(torch.cuda.current_stream(dev))
    return out
