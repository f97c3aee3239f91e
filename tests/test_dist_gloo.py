"""Multi-process (world_size 2, gloo, CPU) coverage of the sharded path.

The per-shard count is injected (the CPU oracle stands in for the sm_100a
kernel, which needs a GPU); the sharding and the allreduce combine are the
product code of paper_2412_16370_b200/dist.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

MIB = 1 << 20


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_count(data, width, counters):
    from oracle import oracle as O
    host = data.numpy() if hasattr(data, "numpy") else np.asarray(data)
    got = O.hs512(host, 0, host.size, width)
    counters[:width] += torch.tensor(got, dtype=torch.int64)


def _worker(rank, world, port, total, width, seed, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2412_16370_b200.dist import pospopcnt_sharded, shard_range
    lo, hi = shard_range(total, world, rank)
    # each rank generates its own slice of the logical array (word_offset)
    full = O.gen_bernoulli(total, seed, q)
    local = torch.from_numpy(full[lo:hi].copy())
    res = pospopcnt_sharded(local, width, count_fn=_oracle_count)
    want = O.hs512(full, 0, total, width)
    assert [int(x) for x in res] == want, (rank, res, want)
    # counters= accumulates into an existing tensor
    acc = torch.ones(width, dtype=torch.int64)
    pospopcnt_sharded(local, width, counters=acc, count_fn=_oracle_count)
    assert [int(x) for x in acc] == [v + 1 for v in want]
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("width,total", [(8, 4 * MIB + 64), (16, 3 * MIB), (64, 2 * MIB + 128)])
def test_sharded_allreduce_gloo_world2(width, total):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, total, width, 0xC5, 30000), nprocs=2, join=True)
