"""Multi-GPU sharding: one process per GPU, counters combined by one allreduce.

The reference is single-threaded by design; counts are
additive over word-complete splits (pkg/tests/test_acceptance.py:
196-204), so a P-way data-parallel count is: contiguous shards cut at
multiples of lcm(16, w/8) bytes, each rank counting its own shard with the
sm_100a kernel, then one ``all_reduce(SUM)`` of the w counters.  Over NCCL on
NVLink/NVSwitch that message is <= 64 x 8 B: latency-bound, a few microseconds.
Counters travel as int64 (identical bits to u64 addition mod 2^64).
"""

import torch
import torch.distributed as dist

from .core import check_width

SHARD_ALIGN = 64  # multiple of 16 (vector) and of every word size


def shard_range(total_bytes, world, rank, align=SHARD_ALIGN):
    """[start, end) of rank's contiguous shard; cuts are multiples of ``align``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    units = total_bytes // align
    lo = units * rank // world * align
    hi = units * (rank + 1) // world * align
    if rank == world - 1:
        hi = total_bytes
    return lo, hi


def _count_cuda(data, width, counters):
    from .kernels import pospopcnt
    return pospopcnt(data, width, counters=counters)


def pospopcnt_sharded(local_data, width, group=None, counters=None, count_fn=None):
    """Count this rank's shard and allreduce the counters over ``group``.

    ``local_data`` is this rank's (word-complete) shard.  Returns an int64
    tensor of ``width`` global counters on the shard's device (added into
    ``counters`` when given).  ``count_fn(data, width, counters_tensor)`` is
    the per-shard counter; it defaults to the sm_100a kernel and exists so
    the collective plumbing can be exercised on CPU with gloo in tests.

    For pipelined jobs (count step i+1 while step i's counters are reduced)
    set ``PP_RESERVE_SMS=8`` before the first count: the persistent counting
    grid then leaves SMs to NCCL's kernels at no cost to its HBM-bound rate.
    """
    check_width(width)
    fn = count_fn or _count_cuda
    dev = local_data.device if hasattr(local_data, "device") else torch.device("cpu")
    local = torch.zeros(width, dtype=torch.int64, device=dev)
    fn(local_data, width, local)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(local, op=dist.ReduceOp.SUM, group=group)
    if counters is not None:
        counters[:width] += local.to(counters.device, counters.dtype)
        return counters
    return local
