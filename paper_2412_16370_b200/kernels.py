"""The B200 kernel object, the registry and the public entry point.

Mirrors the reference's dispatch layer (/root/reference/pkg/src/pospopcnt/
kernels.py:48-63, 276-333): same names (``KERNEL_ENV``, ``list_kernels``,
``get_kernel``, ``select_kernel``, ``pospopcnt``), same error classes, same
accumulate-into-counters contract.  The registry holds exactly one kernel,
``"b200"``, whose ``run`` launches the hand-written sm_100a CUDA kernel
through the C ABI.  It also satisfies the reference's duck-typed kernel
protocol, so ``pospopcnt_ref.pospopcnt(view, w, kernel=B200Kernel())`` works
unchanged (kernels.py:329-333).

Data placement:
  * CUDA tensor, or InputView over one  -> zero-copy, counted in place
  * host bytes / bytearray / memoryview / numpy / CPU tensor
                                        -> pp_count_host: pipelined H2D
                                           copies overlapped with counting
Counter placement:
  * CUDA int64/uint64 tensor (>= w entries) -> accumulated on the device,
    asynchronously on the current stream (no host sync)
  * list / numpy array / anything indexable -> results read back and added
    as Python ints (reference semantics, kernels.py:315-333)
"""

import ctypes
import os
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import (
    InputView,
    KernelUnavailableError,
    UnknownKernelError,
    W_MAX,
    check_width,
    is_torch_tensor,
    new_counters,
)

KERNEL_ENV = "POSPOPCNT_KERNEL"
# host inputs fanned out over several GPUs (pp_count_host_multi): "all" or a
# comma-separated list of CUDA device ordinals; unset = the current device
DEVICES_ENV = "POSPOPCNT_B200_DEVICES"


def _resolve_devices(devices):
    """None | "all" | "0,1,..." | iterable of ints -> tuple of ordinals, or None."""
    if devices is None:
        devices = os.environ.get(DEVICES_ENV) or None
        if devices is None:
            return None
    if isinstance(devices, str):
        if devices.strip().lower() == "all":
            import torch
            n = torch.cuda.device_count()
            if n < 1:
                raise KernelUnavailableError("no CUDA device is visible")
            return tuple(range(n))
        devices = [int(x) for x in devices.split(",") if x.strip()]
    devs = tuple(int(d) for d in devices)
    if not 1 <= len(devs) <= _lib.PP_MAX_FANOUT:
        raise ValueError(f"devices: 1..{_lib.PP_MAX_FANOUT} CUDA device ordinals, got {devs!r}")
    return devs


@dataclass(frozen=True)
class KernelDescriptor:
    """Identity and geometry of a kernel (kernels.py:52-63).

    For the B200 kernel r = 128: each thread's load vector is one 16-byte
    LDS/LDG.128, and block_bytes = 2r as in the reference.
    """

    name: str
    r: int
    block_bytes: int

    def __post_init__(self):
        assert self.r >= W_MAX and self.r & (self.r - 1) == 0


_tls = threading.local()


def _current_stream_handle(torch, dev):
    """The current stream of ``dev`` as a raw cudaStream_t value (the fast
    private accessor when this torch has it: ~1.5 us less per call)."""
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return raw(dev.index)
    return torch.cuda.current_stream(dev).cuda_stream


def _host_u8(base, offset, nbytes):
    """(pointer, keepalive) for a host buffer slice."""
    if is_torch_tensor(base):
        if not base.is_contiguous():
            raise ValueError("input tensor must be contiguous")
        return base.data_ptr() + offset, base
    if isinstance(base, np.ndarray):
        if not base.flags.c_contiguous:
            raise ValueError("input array must be C-contiguous")
        arr = base.reshape(-1).view(np.uint8)
    elif type(base) in (bytes, bytearray):
        arr = np.frombuffer(base, dtype=np.uint8)
    else:
        arr = np.frombuffer(memoryview(base).cast("B"), dtype=np.uint8)
    return arr.__array_interface__["data"][0] + offset, arr


def _device_scratch(device):
    """Per-thread, per-device u64 scratch counters (threads stay independent)."""
    import torch
    cache = getattr(_tls, "scratch", None)
    if cache is None:
        cache = _tls.scratch = {}
    t = cache.get(device)
    if t is None:
        t = cache[device] = torch.zeros(W_MAX, dtype=torch.int64, device=device)
    return t


def _host_result():
    """Per-thread u64[64] host buffer the C calls add results into, zeroed,
    and its address."""
    r = getattr(_tls, "result", None)
    if r is None:
        arr = np.zeros(W_MAX, dtype=np.uint64)
        r = _tls.result = (arr, arr.ctypes.data)
    r[0].fill(0)
    return r


def _device_counters(counters, w, device):
    """counters usable in place on `device`, or None."""
    if is_torch_tensor(counters) and counters.is_cuda:
        import torch
        if counters.device != device:
            raise ValueError("counters live on a different device than the data")
        if counters.dtype not in (torch.int64, torch.uint64) or not counters.is_contiguous():
            raise ValueError("device counters must be a contiguous int64/uint64 tensor")
        return counters
    return None


def _add_into(counters, values, w):
    """counters[j] += values[j] with Python-int semantics (reference contract)."""
    if is_torch_tensor(counters):
        import torch
        counters[:w] += torch.as_tensor(np.asarray(values[:w], dtype=np.int64)).to(
            counters.device, counters.dtype)
        return
    for j, v in enumerate(values[:w].tolist()):  # Python ints in one call
        if v:
            counters[j] += v


class B200Kernel:
    """Hand-written sm_100a positional popcount behind the reference protocol."""

    name = "b200"
    r = 128

    def __init__(self, devices=None, input_ready=False):
        """``devices``: host-resident inputs are split over these GPUs, one
        host link each (pp_count_host_multi); "all", a list of ordinals, or
        None (``POSPOPCNT_B200_DEVICES``, else the current device).  Device
        inputs are always counted where they live.  ``input_ready``: the
        caller vouches that a CUDA input is not written by the kernel queued
        before the count on its stream, so the count's loads may overlap that
        kernel's tail (pp_count_ex, PP_COUNT_INPUT_READY); counter updates
        still wait for it."""
        self.descriptor = KernelDescriptor(self.name, self.r, 2 * self.r)
        self._avail = None
        self.devices = devices
        self.input_ready = bool(input_ready)

    def __repr__(self):
        return f"<kernel {self.name} r={self.r}>"

    def available(self):
        if self._avail is None:
            try:
                info = _lib.device_info(0)
                self._avail = info["cc"][0] == 10
            except Exception:  # noqa: BLE001 - unavailable means unavailable
                self._avail = False
        return self._avail

    def run(self, view, w, counters, fa=None, probe=None):
        """Add the positional popcount of ``view`` into ``counters``.

        Like the reference's compiled kernel (kernels.py:243-244) this
        kernel cannot be instrumented with ``fa`` / ``probe``.
        """
        if fa is not None or probe is not None:
            raise ValueError("the b200 kernel cannot be instrumented")
        check_width(w)
        view = InputView.of(view).check_complete(w)
        if len(counters) < w:
            raise ValueError(f"counter array holds {len(counters)} < {w} entries")
        lib = _lib.load()
        if view.nbytes == 0:
            return counters
        if view.on_device:
            return self._run_device(lib, view, w, counters)
        return self._run_host(lib, view, w, counters)

    def _run_device(self, lib, view, w, counters):
        import torch
        base = view.base
        if not base.is_contiguous():
            raise ValueError("input tensor must be contiguous")
        dev = base.device
        # switch devices only when needed (the context manager costs ~us per call)
        switch = dev.index != torch.cuda.current_device()
        if switch:
            prev = torch.cuda.current_device()
            torch.cuda.set_device(dev)
        try:
            stream = _current_stream_handle(torch, dev)
            ptr = base.data_ptr() + view.offset
            dc = _device_counters(counters, w, dev)
            if dc is not None:
                if self.input_ready:
                    _lib.check(lib.pp_count_ex(ptr, view.nbytes, w, dc.data_ptr(),
                                               _lib.PP_COUNT_INPUT_READY, stream))
                else:
                    _lib.check(lib.pp_count(ptr, view.nbytes, w, dc.data_ptr(), stream))
                return counters
            # host-side counters: count, copy back and synchronise in one C call
            vals, vals_ptr = _host_result()
            _lib.check(lib.pp_count_sync(ptr, view.nbytes, w, vals_ptr, stream))
        finally:
            if switch:
                torch.cuda.set_device(prev)
        _add_into(counters, vals, w)
        return counters

    def _run_host(self, lib, view, w, counters):
        ptr, keep = _host_u8(view.base, view.offset, view.nbytes)
        out, out_ptr = _host_result()
        dev_idx = None
        if is_torch_tensor(counters) and counters.is_cuda:
            dev_idx = counters.device.index
        devs = _resolve_devices(self.devices)
        if devs is not None and (len(devs) > 1 or dev_idx is None):
            arr = (ctypes.c_int * len(devs))(*devs)
            _lib.check(lib.pp_count_host_multi(ptr, view.nbytes, w, out_ptr, arr,
                                               len(devs)))
        elif dev_idx is not None:
            import torch
            with torch.cuda.device(dev_idx):
                _lib.check(lib.pp_count_host(ptr, view.nbytes, w, out_ptr))
        else:
            _lib.check(lib.pp_count_host(ptr, view.nbytes, w, out_ptr))
        del keep
        _add_into(counters, out, w)
        return counters


_KERNELS = None


def _registry():
    """The one built-in kernel (kernels.py:276-285 holds four CPU kernels)."""
    global _KERNELS
    if _KERNELS is None:
        _KERNELS = [B200Kernel()]
    return _KERNELS


def list_kernels():
    """All built-in kernels with availability (kernels.py:288-290)."""
    return [(k.descriptor, k.available()) for k in _registry()]


def get_kernel(name):
    """kernels.py:293-297."""
    for k in _registry():
        if k.name == name:
            return k
    raise UnknownKernelError(f"unknown kernel {name!r}")


def select_kernel(override=None):
    """Resolve a kernel: explicit override, POSPOPCNT_KERNEL, else widest (kernels.py:300-312).

    Unlike the reference there is nothing to fall back to: if no kernel is
    available this raises KernelUnavailableError instead of returning None.
    """
    name = override or os.environ.get(KERNEL_ENV) or None
    if name is not None:
        k = get_kernel(name)
        if not k.available():
            raise KernelUnavailableError(f"kernel {name!r} is not available on this host")
        return k
    best = None
    for k in _registry():
        if k.available() and (best is None or k.r > best.r):
            best = k
    if best is None:
        raise KernelUnavailableError("no pospopcnt kernel is available on this host "
                                     "(needs an sm_100 GPU and libpospopcnt_b200.so)")
    return best


def pospopcnt(data, width, counters=None, kernel=None, *, devices=None, input_ready=False):
    """Add the positional population count of ``data`` to ``counters``.

    Same contract as the reference (kernels.py:315-333): ``data`` is
    bytes-like, a numpy array, a torch tensor (host or CUDA) or an
    InputView over any of these; its length must be a multiple of width/8.
    Returns the counter object (a fresh list when ``counters`` is None).
    ``kernel`` may be a kernel object, a kernel name, or None.
    ``devices`` (keyword only, an extension): split a HOST input over these
    GPUs ("all" or a list of ordinals), one host link each.
    ``input_ready`` (keyword only, an extension): a CUDA input is not
    written by the kernel queued just before this count on its stream, so
    the count's loads may start while that kernel drains (B200Kernel).
    """
    if devices is not None or input_ready:
        if kernel is not None and not (isinstance(kernel, str) and kernel == "b200"):
            raise ValueError("devices= / input_ready= apply to the b200 kernel only")
        kernel = B200Kernel(devices=devices, input_ready=input_ready)
    check_width(width)
    view = InputView.of(data).check_complete(width)
    if counters is None:
        counters = new_counters(width)
    elif len(counters) < width:
        raise ValueError(f"counter array holds {len(counters)} < {width} entries")
    if kernel is None or isinstance(kernel, str):
        kernel = select_kernel(kernel)
    elif not kernel.available():
        raise KernelUnavailableError(f"kernel {kernel.name!r} is not available on this host")
    return kernel.run(view, width, counters)


def fold_frame(frame, w, rot):
    """C_w[j] = sum_{i = j mod w} frame[(i + rot) mod 64]  (flush_fw, accumulate.py:115-130)."""
    return [sum(int(frame[(i + rot) % W_MAX]) for i in range(j, W_MAX, w)) for j in range(w)]


def pospopcnt_all_widths(data, widths=None):
    """Every word width from ONE pass over the data.

    Counts the 64-position address frame once on the GPU (pp_count_frame)
    and folds it for each w in ``widths`` (default: every width the length
    is word-complete for) — the width-refinement identity
    C_w[j] = C_2w[j] + C_2w[j+w] (pkg/tests/test_core.py:66-72).
    Returns {w: list of w counters}.  Host data is copied to the current
    CUDA device once.
    """
    import torch
    view = InputView.of(data)
    if widths is None:
        widths = [w for w in (8, 16, 32, 64) if view.nbytes % (w // 8) == 0]
    for w in widths:
        check_width(w)
        view.check_complete(w)
    lib = _lib.load()
    if view.on_device:
        base, off = view.base, view.offset
    else:
        ptr, keep = _host_u8(view.base, view.offset, view.nbytes)
        host = np.ctypeslib.as_array((ctypes.c_uint8 * view.nbytes).from_address(ptr)) \
            if view.nbytes else np.zeros(0, np.uint8)
        base, off = torch.from_numpy(host.copy()).cuda(), 0
        del keep
    if not base.is_contiguous():
        raise ValueError("input tensor must be contiguous")
    dev = base.device
    frame = np.zeros(W_MAX, dtype=np.uint64)
    ptr = base.data_ptr() + off
    if view.nbytes:
        with torch.cuda.device(dev):
            scratch = _device_scratch(dev)
            scratch.zero_()
            stream = torch.cuda.current_stream(dev).cuda_stream
            _lib.check(lib.pp_count_frame(ptr, view.nbytes, scratch.data_ptr(), stream))
            frame = scratch.cpu().numpy().view(np.uint64)
    rot = 8 * (ptr % 8)
    return {w: fold_frame(frame, w, rot) for w in widths}


def count_device(ptr, nbytes, width, counters_ptr, stream=0, input_ready=False):
    """Raw device-pointer entry (pp_count / pp_count_ex), for callers managing
    their own memory."""
    lib = _lib.load()
    _lib.check(lib.pp_count_ex(ctypes.c_void_p(ptr), nbytes, width, ctypes.c_void_p(counters_ptr),
                               _lib.PP_COUNT_INPUT_READY if input_ready else 0,
                               ctypes.c_void_p(stream)))
