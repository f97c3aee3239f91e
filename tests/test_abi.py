"""The C-ABI library loads and exports every symbol include/*.h declares;
argument validation that needs no device answers with the documented codes."""

import ctypes
import glob
import os
import re

import numpy as np

from paper_2412_16370_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        syms |= set(re.findall(r"^PP_API\s+[\w\s\*]+?\b(pp_\w+)\s*\(", src, re.M))
    return syms


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert {"pp_count", "pp_count_host", "pp_count_segmented", "pp_count_fixed",
            "pp_abi_version", "pp_strerror", "pp_last_error"} <= syms
    assert syms == set(_lib.SIGNATURES), syms ^ set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert getattr(lib, name) is not None, name
    out = os.popen(f"nm -D --defined-only {_lib.LIB_PATH}").read()
    exported = set(re.findall(r"\bT (pp_\w+)", out))
    assert declared_symbols() <= exported
    assert lib.pp_abi_version() == _lib.ABI_VERSION


def test_error_codes_without_device():
    lib = _lib.load()
    buf = np.zeros(64, dtype=np.uint8)
    cnt = np.zeros(64, dtype=np.uint64)
    assert lib.pp_count(buf.ctypes.data, 64, 12, cnt.ctypes.data, None) == _lib.PP_EWIDTH
    assert b"width" in lib.pp_last_error()
    assert lib.pp_count(buf.ctypes.data, 7, 64, cnt.ctypes.data, None) == _lib.PP_ELENGTH
    assert lib.pp_count(buf.ctypes.data, 8, 64, None, None) == _lib.PP_EARG
    assert lib.pp_count_host(buf.ctypes.data, 64, 24, cnt.ctypes.data) == _lib.PP_EWIDTH
    assert lib.pp_count_host(buf.ctypes.data, 3, 16, cnt.ctypes.data) == _lib.PP_ELENGTH
    assert lib.pp_count_host(buf.ctypes.data, 64, 16, None) == _lib.PP_EARG
    # empty host input is a no-op success (core.py:18-20 semantics)
    assert lib.pp_count_host(buf.ctypes.data, 0, 16, cnt.ctypes.data) == _lib.PP_OK
    assert lib.pp_count_fixed(buf.ctypes.data, 3, 4, 16, cnt.ctypes.data, 0, None) == \
        _lib.PP_ELENGTH
    assert lib.pp_count_segmented(buf.ctypes.data, None, 3, 8, cnt.ctypes.data, 0, None) == \
        _lib.PP_EARG
    assert lib.pp_gen_bernoulli(buf.ctypes.data, 64, 1, 0, 70000, None) == _lib.PP_EARG
    devs = (ctypes.c_int * 2)(0, 0)
    assert lib.pp_count_host_multi(buf.ctypes.data, 64, 12, cnt.ctypes.data, devs, 2) == \
        _lib.PP_EWIDTH
    assert lib.pp_count_host_multi(buf.ctypes.data, 3, 16, cnt.ctypes.data, devs, 2) == \
        _lib.PP_ELENGTH
    assert lib.pp_count_host_multi(buf.ctypes.data, 64, 16, cnt.ctypes.data, None, 2) == \
        _lib.PP_EARG
    assert lib.pp_count_host_multi(buf.ctypes.data, 64, 16, cnt.ctypes.data, devs, 0) == \
        _lib.PP_EARG
    stats = np.zeros(4, dtype=np.uint64)
    assert lib.pp_sched_stats(stats.ctypes.data) == _lib.PP_OK
    assert lib.pp_sched_stats(None) == _lib.PP_EARG
    for code in range(6):
        assert lib.pp_strerror(code)
    assert (cnt == 0).all()


def test_error_mapping_to_reference_exceptions():
    import pytest
    import paper_2412_16370_b200 as pp
    lib = _lib.load()
    lib.pp_count(None, 7, 64, None, None)
    with pytest.raises(pp.InputLengthError):
        _lib.check(_lib.PP_ELENGTH)
    with pytest.raises(ValueError):
        _lib.check(_lib.PP_EWIDTH)
    with pytest.raises(pp.KernelUnavailableError):
        _lib.check(_lib.PP_ENODEV)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.PP_ECUDA)


def test_built_for_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out
    sass = os.popen(f"cuobjdump -sass {_lib.LIB_PATH} 2>&1").read()
    # TMA bulk copies + mbarrier pipeline in the counting kernel
    assert "UBLKCP" in sass and "SYNCS" in sass
    assert ctypes.sizeof(ctypes.c_ulonglong) == 8
