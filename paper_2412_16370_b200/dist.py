"""Multi-GPU sharding: one process per GPU, one exchange of <= 64 counters.

The reference is single-threaded by design; counts are
additive over word-complete splits (pkg/tests/test_acceptance.py:
196-204), so a P-way data-parallel count is: contiguous shards cut at
multiples of lcm(16, w/8) bytes, each rank counting its own shard with the
sm_100a kernel, then one sum of the w counters over the ranks.

Two ways to do the sum:

* ``PeerCounters`` (the product path): every rank maps every other rank's
  counter array into its address space once (CUDA IPC; peer access over
  NVLink/NVSwitch), and the counting kernel's epilogue adds each CTA's folded
  counts into ALL ranks' arrays with u64 atomics (``pp_count_multi``).  The
  allreduce is fused into the counting kernel: no collective call per count,
  the exchange overlaps the other CTAs' streaming, and after a barrier every
  rank holds the job total.
* ``all_reduce`` of an int64 tensor over the process group (NCCL, or gloo on
  CPU): the baseline, also what the CPU tests exercise.

Counters travel as int64 (identical bits to u64 addition mod 2^64).
"""

import ctypes

import torch
import torch.distributed as dist

from . import _lib
from .core import W_MAX, check_width

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


class PeerCounters:
    """Every rank's counter arrays, mapped into this process (CUDA IPC).

    Collective constructor: every rank of ``group`` must create one (on its
    own device).  Each rank owns ``NGEN`` int64[64] counter arrays in one
    allocation; the IPC handle of that allocation is exchanged once.

    * generation 0 (``local``) is the raw accumulate-only mode: after every
      rank has run ``count`` over its shard and ``sync()`` has returned,
      ``local`` holds the sum over all ranks' shards, cumulative until
      ``zero()``;
    * generations 1 and 2 serve ``count_call`` (and so
      ``pospopcnt_sharded(peers=...)``): call i counts into generation
      1 + i % 2 of every rank, a barrier waits for every rank's remote adds,
      then each rank reads its own array and zeroes it.  A rank can be at
      most one call ahead of a slower peer (it must pass the next call's
      barrier, which the peer reaches only after its read-and-zero), and
      that call targets the other generation -- so no remote add of a later
      call can land in an array before it is read, and every call returns
      exactly its own job total (the reference's accumulate contract,
      core.py:82-87).
    """

    NGEN = 3

    def __init__(self, group=None, device=None):
        self.lib = _lib.load()
        self.group = group
        self.device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self.gens = torch.zeros((self.NGEN, W_MAX), dtype=torch.int64, device=self.device)
        self.local = self.gens[0]
        self.calls = 0
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        if self.world > _lib.PP_MAX_TARGETS:
            raise ValueError(f"at most {_lib.PP_MAX_TARGETS} ranks per fused exchange")
        handle = ctypes.create_string_buffer(_lib.PP_IPC_HANDLE_BYTES)
        with torch.cuda.device(self.device):
            _lib.check(self.lib.pp_ipc_handle(self.gens.data_ptr(), handle))
        self.handle = handle.raw  # IPC handle of the allocation + offset of `gens` in it
        handles = [handle.raw]
        if self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, handle.raw, group=group)
        self._opened = []
        ptrs = []
        err = None
        with torch.cuda.device(self.device):
            try:
                for r, h in enumerate(handles):
                    if r == self.rank:
                        ptrs.append(self.gens.data_ptr())
                        continue
                    p = ctypes.c_void_p()
                    _lib.check(self.lib.pp_ipc_open(ctypes.create_string_buffer(h, len(h)),
                                                    ctypes.byref(p)))
                    self._opened.append(p.value)
                    ptrs.append(p.value)
            except Exception as exc:  # noqa: BLE001 - agreed on below, then raised
                err = exc
        if self.world > 1:
            # every rank must take the same path: agree on success first
            flag = torch.tensor([0 if err else 1], dtype=torch.int64, device=self.device)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
            if int(flag.item()) == 0 and err is None:
                err = RuntimeError("a peer rank could not map the counter arrays")
        if err is not None:
            self.close()
            raise RuntimeError(f"fused exchange unavailable (no peer mapping): {err}") from err
        # own array first: it is the kernel's primary target
        ptrs.insert(0, ptrs.pop(self.rank))
        row = W_MAX * 8
        self.gen_targets = [(ctypes.c_void_p * len(ptrs))(*[p + g * row for p in ptrs])
                            for g in range(self.NGEN)]
        self.targets = self.gen_targets[0]
        self.sync()

    def count(self, data, nbytes, width, stream=None, gen=0, input_ready=False):
        """Count device bytes [data, data+nbytes) into generation ``gen`` of
        every rank's counters (raw mode: no synchronisation).  ``input_ready``
        as ``pospopcnt`` (pp_count_multi_ex, PP_COUNT_INPUT_READY)."""
        st = torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream
        tg = self.gen_targets[gen]
        flags = _lib.PP_COUNT_INPUT_READY if input_ready else 0
        _lib.check(self.lib.pp_count_multi_ex(ctypes.c_void_p(data), nbytes, width, tg,
                                              len(tg), flags, ctypes.c_void_p(st)))

    def count_call(self, data, nbytes, width):
        """Collective: this call's job total (int64[width], on this rank's
        device) of every rank's shard -- exactly this call's, whatever ran
        before (see the class docstring for the generation protocol)."""
        g = 1 + self.calls % 2
        self.calls += 1
        self.count(data, nbytes, width, gen=g)
        self.sync()  # every rank's remote adds into generation g are complete
        row = self.gens[g]
        out = row[:width].clone()
        row.zero_()
        # the zero must be complete before this rank enters the next call's
        # barrier: peers may add into generation g again one call after that
        torch.cuda.synchronize(self.device)
        return out

    def zero(self):
        """Reset the raw-mode counters (collective: all ranks, before counting)."""
        self.local.zero_()
        self.sync()

    def sync(self):
        """Wait until every rank's pending counts (and so all its remote adds)
        have completed: local device sync + a barrier over the group."""
        torch.cuda.synchronize(self.device)
        if self.world > 1:
            dist.barrier(group=self.group)

    def close(self):
        for p in self._opened:
            self.lib.pp_ipc_close(ctypes.c_void_p(p))
        self._opened = []


def _count_cuda(data, width, counters):
    from .kernels import pospopcnt
    return pospopcnt(data, width, counters=counters)


def pospopcnt_sharded(local_data, width, group=None, counters=None, count_fn=None,
                      peers=None):
    """Count this rank's shard and combine the counters over ``group``.

    ``local_data`` is this rank's (word-complete) shard.  Returns an int64
    tensor of ``width`` global counters on the shard's device (added into
    ``counters`` when given).

    With ``peers`` (a ``PeerCounters``) the combine is fused into the
    counting kernel (remote atomics into every rank's counters over NVLink)
    and only a barrier follows; every call returns (or adds) exactly its own
    job total, like the NCCL path.
    Otherwise the shard is counted into a fresh tensor and all-reduced over
    the group (NCCL, or gloo for CPU tensors).  ``count_fn(data, width,
    counters_tensor)`` replaces the per-shard counter in that path; it exists
    so the collective plumbing can be exercised on CPU with gloo in tests.

    Pipelined NCCL jobs (count step i+1 while step i's counters are reduced)
    should set ``PP_RESERVE_SMS=8`` before the first count: the persistent
    counting grid then leaves SMs to NCCL's kernels at no cost to its
    HBM-bound rate.
    """
    check_width(width)
    if peers is not None:
        from .core import InputView
        view = InputView.of(local_data).check_complete(width)
        if not view.on_device:
            raise ValueError("the fused exchange needs the shard in device memory")
        out = peers.count_call(view.base.data_ptr() + view.offset, view.nbytes, width)
        if counters is not None:
            counters[:width] += out.to(counters.device, counters.dtype)
            return counters
        return out
    fn = count_fn or _count_cuda
    dev = local_data.device if hasattr(local_data, "device") else torch.device("cpu")
    if dev.type != "cuda" and dist.is_available() and dist.is_initialized() and \
            dist.get_backend(group) == "nccl":
        # host-resident shard (counted through pp_count_host): NCCL reduces
        # device tensors only
        dev = torch.device("cuda", torch.cuda.current_device())
    local = torch.zeros(width, dtype=torch.int64, device=dev)
    fn(local_data, width, local)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(local, op=dist.ReduceOp.SUM, group=group)
    if counters is not None:
        counters[:width] += local.to(counters.device, counters.dtype)
        return counters
    return local
