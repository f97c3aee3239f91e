"""The fused allreduce (pp_count_multi through dist.PeerCounters) on one B200.

Two or three processes share cuda:0, exchange CUDA IPC handles of their
counter arrays over gloo, and each counts its own shard with a kernel whose
epilogue adds into EVERY process's counters.  The kernels never wait on one
another (each only issues atomics), so one GPU exercises the real code path:
IPC export/open, the multi-target epilogue, and the barrier protocol.  After
the barrier every rank must hold the oracle count of the whole buffer
(additivity over word-complete shards).
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

MIB = 1 << 20


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, total, lead, width, seed):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from oracle import oracle as O
    from paper_2412_16370_b200.dist import PeerCounters, pospopcnt_sharded, shard_range
    from paper_2412_16370_b200.gen import generate

    # the same logical buffer on every rank, started `lead` bytes into its
    # allocation so the shard addresses exercise flush_fw's rotation
    buf = generate("uniform", (total + lead + 7) // 8 * 8, seed=seed, device="cuda")
    full = buf[lead:lead + total]
    want = O.hs512(full.cpu().numpy(), 0, total, width)
    lo, hi = shard_range(total, world, rank)
    # a small allocation first, so `local` sits inside a caching-allocator
    # block (an interior pointer: its IPC handle must carry the offset)
    pad = torch.empty(4096 + 512 * rank, dtype=torch.uint8, device="cuda")
    peers = PeerCounters(device="cuda:0")
    assert int.from_bytes(peers.handle[64:72], "little") > 0
    del pad
    try:
        got = pospopcnt_sharded(full[lo:hi], width, peers=peers)
        assert [int(x) for x in got.cpu()] == want, (rank, width)
        # every call returns exactly its own job total; counters= adds it
        acc = torch.ones(width, dtype=torch.int64, device="cuda")
        pospopcnt_sharded(full[lo:hi], width, peers=peers, counters=acc)
        assert [int(x) for x in acc.cpu()] == [v + 1 for v in want], (rank, width)
        got = pospopcnt_sharded(full[lo:hi], width, peers=peers)
        assert [int(x) for x in got.cpu()] == want, (rank, width)
        # reset and count a second, uneven split: ranks' kernels race freely
        peers.zero()
        cut = [0, total // 3 // 8 * 8, total]
        if world == 2:
            part = full[cut[rank]:cut[rank + 1]]
        else:
            part = full[lo:hi]
        for i in range(3):  # the buffer is written before any count: input_ready holds
            peers.count(part.data_ptr(), part.numel(), width, input_ready=bool(i % 2))
        peers.sync()
        assert [int(x) for x in peers.local[:width].cpu()] == [3 * v for v in want]
        # an empty shard is fine (its CTAs add zeros)
        peers.zero()
        peers.count(full.data_ptr(), total if rank == 1 else 0, width)
        peers.sync()
        assert [int(x) for x in peers.local[:width].cpu()] == want
    finally:
        dist.barrier()
        peers.close()
        dist.destroy_process_group()


@pytest.mark.parametrize("world,width,total,lead", [
    (2, 8, 64 * MIB + 24, 3),
    (2, 16, 17 * MIB + 6, 2),
    (2, 32, 8 * MIB + 4, 4),
    (2, 64, 40 * MIB + 8, 0),
    (3, 8, 33 * MIB + 1, 5),
    (3, 64, 3 * MIB + 72, 8),
])
def test_fused_exchange_one_gpu(cuda, world, width, total, lead):
    mp.spawn(_worker, args=(world, _free_port(), total, lead, width, 0xF5ED + width),
             nprocs=world, join=True)


def _calls_worker(rank, world, port, ncalls, seed):
    """ncalls back-to-back sharded calls over tiny, uneven shards, nothing
    zeroed in between: ranks race through the calls at different speeds
    (rank r sleeps r-dependent amounts), and every call must return exactly
    that call's job total (dist.PeerCounters generation protocol)."""
    import sys
    import time
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import numpy as np
    from oracle import oracle as O
    from paper_2412_16370_b200.dist import PeerCounters, pospopcnt_sharded

    rng = np.random.default_rng(seed)
    peers = PeerCounters(device="cuda:0")
    try:
        for i in range(ncalls):
            width = (8, 16, 32, 64)[i % 4]
            # the same per-call data on every rank (seeded by the call index)
            host = np.random.default_rng(seed + i).integers(0, 256, 4096 + 64 * (i % 7),
                                                             dtype=np.uint8)
            want = O.hs512(host, 0, host.size, width)
            cut = (host.size // world) // 8 * 8
            lo, hi = rank * cut, (host.size if rank == world - 1 else (rank + 1) * cut)
            shard = torch.from_numpy(host[lo:hi].copy()).cuda()
            if rng.random() < 0.3:
                time.sleep(0.002 * (rank + 1))
            got = pospopcnt_sharded(shard, width, peers=peers)
            assert [int(x) for x in got.cpu()] == want, (rank, i, width)
    finally:
        dist.barrier()
        peers.close()
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_exchange_per_call_totals(cuda, world):
    mp.spawn(_calls_worker, args=(world, _free_port(), 200, 0xCA11), nprocs=world, join=True)


def test_multi_rejects_bad_targets(cuda):
    import ctypes
    from paper_2412_16370_b200 import _lib
    lib = _lib.load()
    data = torch.zeros(1024, dtype=torch.uint8, device="cuda")
    ctr = torch.zeros(64, dtype=torch.int64, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    none = (ctypes.c_void_p * 1)()
    assert lib.pp_count_multi(data.data_ptr(), 1024, 8, none, 0, st) == _lib.PP_EARG
    too_many = (ctypes.c_void_p * 17)(*([ctr.data_ptr()] * 17))
    assert lib.pp_count_multi(data.data_ptr(), 1024, 8, too_many, 17, st) == _lib.PP_EARG
    host = (ctypes.c_uint64 * 64)()
    bad = (ctypes.c_void_p * 2)(ctr.data_ptr(), ctypes.addressof(host))
    assert lib.pp_count_multi(data.data_ptr(), 1024, 8, bad, 2, st) != _lib.PP_OK
    # the same array twice is legal: it receives the counts twice
    data.fill_(0xFF)
    twice = (ctypes.c_void_p * 2)(ctr.data_ptr(), ctr.data_ptr())
    assert lib.pp_count_multi(data.data_ptr(), 1024, 8, twice, 2, st) == _lib.PP_OK
    torch.cuda.synchronize()
    assert ctr[:8].tolist() == [2048] * 8


def test_sharded_host_shard_over_nccl(cuda, oracle):
    """pospopcnt_sharded on a host-resident shard with the NCCL backend (one
    rank): the shard goes through pp_count_host, the counters are reduced
    as a device tensor."""
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    child = (
        "import sys, numpy as np, torch, torch.distributed as dist\n"
        f"sys.path.insert(0, {root!r})\n"
        "from oracle import oracle as O\n"
        "from paper_2412_16370_b200.dist import pospopcnt_sharded\n"
        "torch.cuda.set_device(0)\n"
        f"dist.init_process_group('nccl', init_method='tcp://127.0.0.1:{port}', rank=0,"
        " world_size=1, device_id=torch.device('cuda', 0))\n"
        "host = np.random.default_rng(2).integers(0, 256, (40 << 20) + 8, dtype=np.uint8)\n"
        "got = pospopcnt_sharded(host.tobytes(), 64)\n"
        "assert got.is_cuda and [int(x) for x in got.cpu()] == O.hs512(host, 0, host.size, 64)\n"
        "dist.destroy_process_group()\n"
        "print('ok')\n")
    res = subprocess.run([sys.executable, "-c", child], capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0 and res.stdout.strip().endswith("ok"), res.stdout + res.stderr
