"""pp_count_host_multi: one call over a host buffer fanned out over several
GPUs, one host link (staging ring + copy stream) per listed device.

The box has one GPU, so the fan-out logic -- the 64-byte range cuts, one
persistent worker per listing, per-worker staging contexts and the host-side
sum -- is exercised by listing cuda:0 several times; the ranges then share a
link but every code path is the multi-device one.  Expected counts come from
the CPU oracle (C restatement of the reference, oracle/)."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MIB = 1 << 20


@pytest.mark.parametrize("ndev", [1, 2, 3, 8])
@pytest.mark.parametrize("nbytes,width", [
    (0, 8), (8, 64), (64, 16), (64 * 3 + 8, 64), (1000, 8), (MIB + 40, 32),
    (96 * MIB + 24, 64), (129 * MIB + 2, 16),
])
def test_fanout_matches_oracle(cuda, oracle, ndev, nbytes, width):
    import paper_2412_16370_b200 as pp
    host = np.random.default_rng(nbytes + ndev).integers(0, 256, nbytes, dtype=np.uint8)
    want = oracle.hs512(host, 0, nbytes, width)
    got = pp.pospopcnt(host, width, devices=[0] * ndev)
    assert [int(x) for x in got] == want
    # accumulate contract: a second call adds
    got = pp.pospopcnt(host, width, counters=got, devices=[0] * ndev)
    assert [int(x) for x in got] == [2 * v for v in want]


def test_fanout_pinned_and_pageable(cuda, oracle):
    torch, pp = cuda
    n = 200 * MIB + 64
    pinned = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    pinned.random_(0, 256, generator=torch.Generator().manual_seed(7))
    host = pinned.numpy()
    want = oracle.hs512(host, 0, n, 8, threads=8)
    assert [int(x) for x in pp.pospopcnt(pinned, 8, devices="0,0,0,0")] == want
    assert [int(x) for x in pp.pospopcnt(host.tobytes(), 8, devices=[0, 0])] == want
    # the kernel object carries the device list through the reference protocol
    k = pp.B200Kernel(devices=[0, 0, 0])
    assert [int(x) for x in pp.pospopcnt(pp.InputView(pinned, 3, n - 67), 8, kernel=k)] == \
        oracle.hs512(host, 3, n - 67, 8, threads=8)


def test_fanout_rejects_bad_devices(cuda):
    torch, pp = cuda
    from paper_2412_16370_b200 import _lib
    lib = _lib.load()
    buf = np.zeros(4096, dtype=np.uint8)
    out = np.zeros(64, dtype=np.uint64)
    bad = (ctypes.c_int * 2)(0, torch.cuda.device_count())
    assert lib.pp_count_host_multi(buf.ctypes.data, 4096, 8, out.ctypes.data, bad, 2) == \
        _lib.PP_EARG
    assert lib.pp_count_host_multi(buf.ctypes.data, 4096, 8, out.ctypes.data, None, 1) == \
        _lib.PP_EARG
    many = (ctypes.c_int * 17)(*([0] * 17))
    assert lib.pp_count_host_multi(buf.ctypes.data, 4096, 8, out.ctypes.data, many, 17) == \
        _lib.PP_EARG
    dev_buf = torch.zeros(4096, dtype=torch.uint8, device="cuda")
    one = (ctypes.c_int * 1)(0)
    assert lib.pp_count_host_multi(dev_buf.data_ptr(), 4096, 8, out.ctypes.data, one, 1) == \
        _lib.PP_EARG
    with pytest.raises(ValueError):
        pp.pospopcnt(buf, 8, devices=[])
    assert not out.any()
