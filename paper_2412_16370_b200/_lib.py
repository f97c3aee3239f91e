"""ctypes binding of libpospopcnt_b200.so (include/pospopcnt_b200.h).

The library is built in-tree by ``paper_2412_16370_b200.build``.  If it is
missing or cannot be loaded, every entry point raises KernelUnavailableError:
there is no CPU fallback anywhere in this package.  ctypes releases the GIL
for the duration of each call.
"""

import ctypes
import os
import threading

from .core import InputLengthError, KernelUnavailableError

HERE = os.path.dirname(os.path.abspath(__file__))
# PP_LIB_PATH: load an alternative build (A/B experiments, scripts/)
LIB_PATH = os.environ.get("PP_LIB_PATH") or os.path.join(HERE, "libpospopcnt_b200.so")

PP_OK, PP_EWIDTH, PP_ELENGTH, PP_ECUDA, PP_EARG, PP_ENODEV = range(6)
PP_SEG_ACCUMULATE, PP_SEG_OVERWRITE = 0, 1
PP_SEG_HYBRID = 1 << 16    # CSR: <= 512 B arrays one lane each, the rest G lanes
PP_SEG_BATCH_SHIFT = 20    # PP_SEG_BATCH(t): groups per scheduler ticket hint (0 = auto)
PP_MAX_TARGETS = 16        # pp_count_multi: counter arrays per call
PP_MAX_FANOUT = 16         # pp_count_host_multi: devices per call
PP_IPC_HANDLE_BYTES = 72   # pp_ipc_handle: CUDA IPC handle + offset in the allocation
ABI_VERSION = 1
PP_COUNT_INPUT_READY = 1   # pp_count_ex: loads need not wait for the previous kernel

# name -> (restype, argtypes); mirrors include/pospopcnt_b200.h
_vp, _sz, _int, _u64, _u32 = (ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                               ctypes.c_uint64, ctypes.c_uint32)
SIGNATURES = {
    "pp_abi_version": (_int, []),
    "pp_strerror": (ctypes.c_char_p, [_int]),
    "pp_last_error": (ctypes.c_char_p, []),
    "pp_device_info": (_int, [_int, _vp, _vp, _vp]),
    "pp_count": (_int, [_vp, _sz, _int, _vp, _vp]),
    "pp_count_ex": (_int, [_vp, _sz, _int, _vp, _u32, _vp]),
    "pp_count_host": (_int, [_vp, _sz, _int, _vp]),
    "pp_count_sync": (_int, [_vp, _sz, _int, _vp, _vp]),
    "pp_count_host_multi": (_int, [_vp, _sz, _int, _vp, _vp, _int]),
    "pp_sched_stats": (_int, [_vp]),
    "pp_check_status": (_int, [_vp, _int]),
    "pp_debug_corrupt": (_int, [_int]),
    "pp_count_frame": (_int, [_vp, _sz, _vp, _vp]),
    "pp_count_multi": (_int, [_vp, _sz, _int, _vp, _int, _vp]),
    "pp_count_multi_ex": (_int, [_vp, _sz, _int, _vp, _int, _u32, _vp]),
    "pp_ipc_handle": (_int, [_vp, _vp]),
    "pp_ipc_open": (_int, [_vp, _vp]),
    "pp_ipc_close": (_int, [_vp]),
    "pp_count_categories": (_int, [_vp, _sz, _int, _int, _vp, _vp]),
    "pp_count_categories_ex": (_int, [_vp, _sz, _int, _int, _vp, _u32, _vp]),
    "pp_count_segmented": (_int, [_vp, _vp, _sz, _int, _vp, _int, _vp]),
    "pp_count_segmented_order": (_int, [_vp, _vp, _vp, _sz, _int, _vp, _int, _vp]),
    "pp_count_fixed": (_int, [_vp, _sz, _sz, _int, _vp, _int, _vp]),
    "pp_count_batch": (_int, [_vp, _vp, _sz, _int, _vp, _int, _vp]),
    "pp_readonly_sum": (_int, [_vp, _sz, _vp, _vp]),
    "pp_readonly_sum_ex": (_int, [_vp, _sz, _vp, _u32, _vp]),
    "pp_gen_uniform": (_int, [_vp, _sz, _u64, _u64, _vp]),
    "pp_gen_bernoulli": (_int, [_vp, _sz, _u64, _u64, _u32, _vp]),
    "pp_gen_blocks": (_int, [_vp, _sz, _u64, _u64, _u64, _vp]),
    "pp_gen_onehot32": (_int, [_vp, _sz, _u64, _u64, _vp, _vp]),
    "pp_gen_codes8": (_int, [_vp, _sz, _u64, _u64, _vp, _vp]),
}

_lock = threading.Lock()
_lib = None
_load_error = None


def load():
    """Load (building first if absent) and type the shared library."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if _load_error is not None:
            raise KernelUnavailableError(_load_error)
        try:
            if not os.path.exists(LIB_PATH):
                from . import build as _build
                _build.build()
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                try:
                    f = getattr(lib, name)
                except AttributeError:
                    if os.environ.get("PP_LIB_PATH"):
                        continue  # an older A/B build: only its own entry points
                    raise
                f.restype = res
                f.argtypes = args
            if lib.pp_abi_version() != ABI_VERSION:
                raise RuntimeError("ABI version mismatch")
        except Exception as exc:  # noqa: BLE001 - reported loudly below
            _load_error = f"libpospopcnt_b200.so unavailable: {exc}"
            raise KernelUnavailableError(_load_error) from exc
        _lib = lib
        if os.environ.get("PP_CHECK_REPORT"):
            import atexit
            atexit.register(_check_report, os.environ["PP_CHECK_REPORT"])
        return _lib


def check_status(reset=False):
    """pp_check_status as a dict (checked builds: PP_CHECK_BOUNDS=1)."""
    out = (ctypes.c_uint64 * 6)()
    check(load().pp_check_status(out, 1 if reset else 0))
    return {"checked_build": bool(out[0]), "fails": int(out[1]), "first_line": int(out[2]),
            "first_addr": int(out[3]), "first_lo": int(out[4]), "first_hi": int(out[5])}


def _check_report(path):
    """PP_CHECK_REPORT=<file>: at exit, append this process's check record
    (the tests running a checked build collect one line per process)."""
    try:
        st = check_status()
        with open(path, "a") as f:
            f.write(f"{os.getpid()} {int(st['checked_build'])} {st['fails']} {st['first_line']} "
                    f"{st['first_addr']:#x} {st['first_lo']:#x} {st['first_hi']:#x}\n")
    except Exception as exc:  # noqa: BLE001 - reported as a failed record
        with open(path, "a") as f:
            f.write(f"{os.getpid()} error {exc!r}\n")


def check(rc):
    """Map a PP_E* return code to the reference's exception classes."""
    if rc == PP_OK:
        return
    msg = (_lib.pp_last_error() or b"").decode() or _lib.pp_strerror(rc).decode()
    if rc == PP_ELENGTH:
        raise InputLengthError(msg)
    if rc in (PP_EWIDTH, PP_EARG):
        raise ValueError(msg)
    if rc == PP_ENODEV:
        raise KernelUnavailableError(msg)
    raise RuntimeError(msg)


def device_info(device=0):
    lib = load()
    sms, ma, mi = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    check(lib.pp_device_info(device, ctypes.byref(sms), ctypes.byref(ma), ctypes.byref(mi)))
    return {"num_sms": sms.value, "cc": (ma.value, mi.value)}
