#!/usr/bin/env python3
"""Benchmark of the B200 positional population count (driver contract).

Default (N=1): BASELINE.json configs[1] = C2, w=8 over a 1 GiB array of
Bernoulli(0.5) bits generated in place in HBM.  One step = one pass of the
hot path (pp_count, one launch of the sm_100a kernel) over the whole array.
Under torchrun (any N) each rank counts its own 1 GiB shard of an N GiB
array (weak scaling); by default the counter exchange is fused into the
counting kernel (``pp_count_multi`` adds every CTA's counts into all ranks'
IPC-mapped counters, no collective per step); ``--exchange nccl`` instead
allreduces each step's counters over NCCL, pipelined on a side stream.
``--config c5`` is the fixed 64 GiB array split over the N ranks (strong
scaling).

Printed JSON keys beyond the base contract:
  roofline       dominant kernel: algorithmic bytes per launch (n input bytes,
                 SURVEY.md 8d) / mean launch time vs MEASURED_PEAKS.hbm_gbs,
                 plus the in-run read-only roofline kernel and ncu traffic
  cpu_baseline   the reference's fastest CPU path on the host's cores, bounded
                 sample: the unmodified reference (baseline/_ref, numba kernel
                 on P forked processes) when it is installed, else the C
                 restatement of NumbaKernel.run (oracle/)
  e2e            the same metric through the public API pospopcnt() on a
                 pinned HOST buffer: H2D copies + D2H of the counters inside
                 the timed region; e2e_pageable: the same call on a pageable
                 numpy array; e2e_fanout: one host buffer over every GPU
  exact          counters after all steps == steps x expected (CPU oracle, or
                 the reference's own golden totals for C3 codes / C5)
  per_width_gbs  C2 bytes counted at every word width (the metric is per w)
  clocks         NVML SM clock / throttle reasons sampled inside the region

``--impl reference`` times the reference's CPU implementation (the unmodified
reference from baseline/_ref on all host cores; the oracle's C port only when
that install is absent) on the same config.  ``--config`` selects another config (c1, c3,
c3cat, c4, c4seg, c5) for an extra line.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pospopcnt input GB/s (fraction of HBM peak) at 1/2/4/8 B200, per word width"
GIB = 1 << 30
MIB = 1 << 20
SPEC_HBM_GBS = 7700.0  # B200 HBM3e datasheet bandwidth (HGX figure; B200_PROFILING.md)
SETTLE_MS = 30.0
L2_FLUSH_BELOW = 256 * MIB  # inputs below this may stay in the 126 MB L2: flush per step
L2_FLUSH_BYTES = 512 * MIB  # untimed device work after the W warm-up steps (see main_gpu)

CONFIGS = {
    # name: (generator, width, bytes per GPU (weak) or in total (strong), description)
    "c1": ("uniform", 16, 2 * MIB, "w=16, 2 MiB, Bernoulli(0.5), aligned"),
    "c2": ("uniform", 8, GIB, "w=8, 1 GiB, Bernoulli(0.5)"),
    "c3": ("onehot32", 32, 4 * GIB, "w=32 one-hot, 4 GiB, bounded Zipf(1.1) over 32 bits"),
    "c4": ("bernoulli", 64, 64 * MIB, "w=64, 64 MiB at byte offset 3, Bernoulli(0.01)"),
    "c4seg": ("bernoulli", 64, GIB, "w=64, 262,144 segments x 4 KiB, Bernoulli(0.01)"),
    "c3cat": ("codes8", 32, GIB, "w=32 GROUP BY COUNT: 2^30 u8 category codes with C3's Zipf "
                                  "draws, fused one-hot producer (pp_count_categories)"),
    "c5": ("blocks", 16, 64 * GIB, "w=16, 64 GiB array sharded over the GPUs (8 GiB per GPU "
                                   "at N=8), Bernoulli(p) with p ~ U[0,1] per 1 MiB block"),
}
STRONG = {"c5"}  # total work fixed as N grows; every other config is per-GPU (weak)


def golden_total(name):
    """The reference's own counters for a full config (tests/golden/golden.json)."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
            return json.load(f)["digests"][name]["expected"]
    except Exception:  # noqa: BLE001
        return None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def load_traffic(kernel_key, input_bytes):
    """(dram bytes per launch, dram bytes per input byte) of the dominant kernel
    from the committed ncu capture; the absolute figure only when the capture
    counted a launch of the same input size as this one."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)[kernel_key]
        ratio = d["bytes"] / d["input_bytes"]
        return (d["bytes"] if d["input_bytes"] == input_bytes else None), round(ratio, 5)
    except Exception:  # noqa: BLE001
        return None, None


def load_alu(kernel_key):
    """(ALU-pipe lane-instructions, shared-memory wavefronts) per input byte
    (= per u8 code) of a fused producer kernel, from the committed ncu
    capture (profiles/ncu_alu.json); None where absent."""
    p = os.path.join(ROOT, "profiles", "ncu_alu.json")
    try:
        with open(p) as f:
            d = json.load(f)[kernel_key]
        alu = round(d["alu_warp_inst"] * 32 / d["input_bytes"], 4)
        lds = d.get("lds_wavefronts")
        return alu, (lds / d["input_bytes"] if lds else None)
    except Exception:  # noqa: BLE001
        return None, None


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, ~1 ms period) while the
    timed region runs; mark() brackets the region on the host clock.  Falls
    back to one nvidia-smi query per sample if NVML is unavailable."""

    REASONS = {  # NVML clocks-event-reason bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap",
    }

    def __init__(self, index, period=None):
        period = float(os.environ.get("PP_BENCH_CLOCK_PERIOD", "0.001")) if period is None else period
        self.index, self.period = index, period
        self.samples = []  # (t, sm_mhz, reasons_mask)
        self.t0 = self.t1 = None
        self.stop = threading.Event()
        self.max_mhz = None
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = None
            try:  # CUDA ordinal -> NVML handle via the PCI bus id (CUDA_VISIBLE_DEVICES-safe)
                import torch
                pr = torch.cuda.get_device_properties(self.index)
                dom, bus, devn = (int(pr.pci_domain_id), int(pr.pci_bus_id),
                                  int(pr.pci_device_id))
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(
                    f"{dom:08X}:{bus:02X}:{devn:02X}.0")
            except Exception:  # noqa: BLE001
                self.h = None
            if self.h is None:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nvml = None
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        return self

    def _sample(self):
        if self.nvml is not None:
            p = self.nvml
            return (p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM),
                    p.nvmlDeviceGetCurrentClocksEventReasons(self.h))
        out = subprocess.run(
            ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm",
             "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout
        sm, mx = (float(x) for x in out.strip().split(","))
        self.max_mhz = mx
        return sm, 0

    def _run(self):
        while not self.stop.is_set():
            try:
                sm, mask = self._sample()
                self.samples.append((time.perf_counter(), sm, mask))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def mark(self, start):
        if start:
            self.t0 = time.perf_counter()
        else:
            self.t1 = time.perf_counter()

    def __exit__(self, *exc):
        self.stop.set()
        self.th.join(timeout=2)

    def summary(self):
        inside = [s for s in self.samples
                  if self.t0 is not None and self.t1 is not None and self.t0 <= s[0] <= self.t1]
        window = "timed region"
        if not inside:  # region shorter than one sample period: nearest samples
            inside = sorted(self.samples, key=lambda s: abs(s[0] - (self.t0 or 0)))[:3]
            window = "nearest samples to the timed region"
        reasons = set()
        for _, _, mask in inside:
            for bit, name in self.REASONS.items():
                if mask & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median([s[1] for s in inside]) if inside else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(inside), "window": window,
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def gpu_busy(ms=1.0):
    """Queue a ~ms spin kernel on the current stream before a start event, so
    the timed launches are already queued when the event fires (the timed
    region then measures device throughput, not host launch latency)."""
    import torch
    torch.cuda._sleep(int(ms * 2.0e6))  # ~2e6 cycles per ms at ~2 GHz


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


# ------------------------------------------------------------ CPU legs

def config_dict(cfg, world, per_gpu_bytes, job_bytes, w):
    """The workload description both arms print (identical dicts, so the
    driver can match the reference arm's line to this arm's)."""
    kind, w0, _, desc = CONFIGS[cfg]
    if w != w0:  # --width override of C2's word width
        desc = desc.replace(f"w={w0},", f"w={w},", 1)
    if cfg == "c4seg":
        par = f"dp{world} (segment ranges; rows stay on their rank, no exchange)"
    else:
        par = (f"dp{world} (contiguous 64-byte-cut shards; the {w} counters combined by the "
               "counting kernel's fused peer exchange, NCCL allreduce fallback)")
    return {"workload": desc, "word_width": w, "bytes_per_gpu_per_step": per_gpu_bytes,
            "bytes_per_step_all_gpus": job_bytes,
            "parallelism": par if world > 1 else "single GPU"}


def host_sample(cfg, nbytes):
    """The config's bytes (same generators and seeds as the GPU arm) for the
    CPU legs; returns (u8 array, unit_bytes, w, seg)."""
    from oracle import oracle as O  # bench's cpu_baseline leg: data generation only
    kind, w, _, _ = CONFIGS[cfg]
    unit_bytes, seg = 1, 0
    if kind == "uniform":
        host = O.gen_uniform(nbytes, 0xC2 if cfg == "c2" else 0xC1)
    elif kind == "onehot32":
        host = O.gen_onehot32(nbytes, 0xC3)
    elif kind == "codes8":
        # the reference counts categories as one-hot words:
        # 4 bytes of one-hot u32 per code; the metric is per code byte
        host = O.gen_onehot32(nbytes, 0xC3)
        unit_bytes = 4
    elif kind == "bernoulli":
        host = O.gen_bernoulli(nbytes, 0xC4 + (1 if cfg == "c4seg" else 0), 655)
        seg = 4096 if cfg == "c4seg" else 0
    else:
        host = O.gen_blocks(nbytes, 0xC5)
    return host, unit_bytes, w, seg


def cpu_leg(cfg, sample_bytes, min_time, with_rows=True):
    """The reference's CPU path on this host: the installed reference's numba
    kernel on P forked processes (kind "reference"), else the C port on P
    threads (kind "port").  Returns the cpu_baseline object."""
    import bench_cpu as BC
    host, unit_bytes, w, seg = host_sample(cfg, sample_bytes)
    ref, why = BC.load_reference()
    info = BC.host_info()
    what = f"{host.size >> 20} MiB of the {cfg} array" + (
        " (one-hot u32 words of the codes)" if unit_bytes == 4 else "") + (
        " as 4 KiB arrays, one reference call each" if seg else "")
    if ref is not None:
        # calibrate: steps so one timed run lasts >= min_time
        k, t = 2, 0.0
        for _ in range(4):  # k grows until one timed run lasts >= min_time
            t, _, procs = BC.run_ref_pcore(host, w, k, 1, seg=seg)
            if t >= min_time:
                break
            k = max(k + 1, int(k * min_time / max(t, 1e-6) * 1.1) + 1)
        gbs = host.size / unit_bytes * k / t / 1e9
        out = {"value": round(gbs, 3), "unit": "GB/s", "cores": procs, "kind": "reference",
               "sample": f"{what}, {k} passes in {t:.2f} s on {procs} forked processes: the "
                         "unmodified reference (baseline/_ref) pospopcnt(InputView, w, "
                         "kernel='numba') (kernels.py:315-333, 218-270) over contiguous "
                         "64-byte-cut shards",
               "host": info}
        if with_rows:
            rows = BC.ref_rows(host[: min(host.size, 256 << 20)], w, min_time=min(2.0, min_time),
                               scalar=cfg in ("c1", "c2"))
            rows["ref-numba-Pcore"] = {"GBs": out["value"], "cores": procs}
            out["rows"] = rows
            out["one_core"] = rows.get("ref-numba-1core", {}).get("GBs")
        return out
    gbs, threads, _, k, t = BC.port_pcore(host, w, min_time, seg=seg)
    gbs /= unit_bytes
    return {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"{what}, counted {k}x in {t:.1f} s (last of >=2 rounds); C restatement "
                      f"of NumbaKernel.run (kernels.py:242-270, oracle/) on {threads} host "
                      f"threads -- the reference itself is unavailable: {why}",
            "host": info}


def run_reference(args):
    """--impl reference: the reference's CPU path on the host cores, same
    config, metric and unit as the GPU arm; rank 0 only under torchrun."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import bench_cpu as BC
    cfg = args.config
    kind, w, nbytes, desc = CONFIGS[cfg]
    world = args.gpus or int(os.environ.get("WORLD_SIZE", "1"))
    per_gpu = nbytes if cfg not in STRONG else nbytes // world
    job = per_gpu * world if cfg not in STRONG else nbytes
    sample = min(nbytes, GIB)  # bounded sample of the workload (the metric is a rate)
    host, unit_bytes, w, seg = host_sample(cfg, sample)
    ref, why = BC.load_reference()
    if ref is not None:
        t, _, procs = BC.run_ref_pcore(host, w, args.steps, args.warmup, seg=seg)
        impl_kind = "reference"
        impl_desc = ("the unmodified reference (baseline/_ref) pospopcnt(InputView, w, "
                     "kernel='numba') (kernels.py:315-333, 218-270) on "
                     f"{procs} forked processes over contiguous 64-byte-cut shards")
    else:
        import numpy as np
        from oracle import oracle as O
        procs = BC.host_threads()
        if seg:
            offs = np.arange(host.size // seg + 1, dtype=np.uint64) * seg
            run = lambda: O.segments(host, offs, w, threads=procs)  # noqa: E731
        else:
            run = lambda: O.hs512(host, 0, host.size, w, threads=procs)  # noqa: E731
        for _ in range(args.warmup):
            run()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            run()
        t = time.perf_counter() - t0
        impl_kind = "port"
        impl_desc = (f"C restatement of NumbaKernel.run (kernels.py:242-270, oracle/) on {procs} "
                     f"threads; the reference itself is unavailable: {why}")
    value = host.size / unit_bytes * args.steps / t / 1e9
    line = {
        "impl": "reference",
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * t / args.steps, 3), "higher_is_better": True,
        "scaling": "strong" if cfg in STRONG else "weak", "vs_baseline": None,
        "dtype": "u8" if w == 8 else f"u{w}",
        "data": "synthetic: seeded splitmix64 generators (the GPU arm's bytes)",
        "config": config_dict(cfg, world, per_gpu, job, w),
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": procs,
                         "kind": impl_kind,
                         "sample": f"a {host.size >> 20} MiB sample of the {cfg} workload per "
                                   "step" + (" (one-hot u32 words of the codes)"
                                             if unit_bytes == 4 else "") + "; " + impl_desc,
                         "host": BC.host_info()},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    emit(line)
    return 0


# ------------------------------------------------------------ GPU arm

def sm100_devices():
    """Ordinals of the visible sm_100 devices."""
    import torch
    return [i for i in range(torch.cuda.device_count())
            if torch.cuda.get_device_capability(i)[0] == 10]


def require_devices(n, local=None):
    """Fail loudly unless n sm_100 devices are visible (and this rank's is one)."""
    devs = sm100_devices()
    if len(devs) < n or (local is not None and local not in devs):
        raise SystemExit(f"bench.py: {n} rank(s) need {n} visible sm_100 GPUs; visible sm_100 "
                         f"devices: {devs}")


def bind_to_gpu_numa_node(local):
    """Pin this rank's host threads to the CPUs NVML names as closest to its
    GPU (N > 1 only): the rank's pinned host buffers are then first-touched
    on the GPU's own NUMA node, so N ranks' host->device copies do not all
    cross the socket interconnect.  Returns the CPU count, or None."""
    try:
        import pynvml
        import torch
        uuid = str(torch.cuda.get_device_properties(local).uuid)
        pynvml.nvmlInit()
        try:
            h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        finally:
            pynvml.nvmlShutdown()
        cpus = {64 * i + b for i, wd in enumerate(words) for b in range(64) if (wd >> b) & 1}
        cpus &= set(range(os.cpu_count() or 1))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception as exc:  # noqa: BLE001 - an optimisation, never a failure
        print(f"bench: no NUMA binding ({exc})", file=sys.stderr)
    return None


def run_strong_c5(args, lib, world, rank, dev, st, use_dist, peers):
    """C5 (BASELINE.json configs[4]): the 64 GiB w=16 array with p ~ U[0,1]
    per 1 MiB block, split over the N ranks in contiguous 64-byte-cut shards
    generated in place; every step counts each rank's shard and combines the
    16 counters over the ranks (the fused in-kernel exchange when mapped,
    else an NCCL allreduce per step inside the timed region).  The job total
    after all steps must equal steps x the reference's own 64 GiB total."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2412_16370_b200 import _lib, gen
    from paper_2412_16370_b200.dist import shard_range
    total, w = CONFIGS["c5"][2], 16
    lo, hi = shard_range(total, world, rank)
    shard = gen.generate("blocks", hi - lo, 0xC5, device=dev, word_offset=lo // 8)
    ptr, n = shard.data_ptr(), hi - lo
    ctr = torch.zeros(64, dtype=torch.int64, device=dev)
    fused = peers is not None
    if fused:
        peers.zero()

    def step():
        if fused:
            _lib.check(lib.pp_count_multi(ptr, n, w, peers.targets, len(peers.targets),
                                          st.cuda_stream))
        elif use_dist:  # this step's shard counts, reduced, added to the job total
            ctr.zero_()
            _lib.check(lib.pp_count(ptr, n, w, ctr.data_ptr(), st.cuda_stream))
            dist.all_reduce(ctr)
            glob.add_(ctr)
        else:
            _lib.check(lib.pp_count(ptr, n, w, ctr.data_ptr(), st.cuda_stream))
    glob = torch.zeros(64, dtype=torch.int64, device=dev)
    warm, steps = 2, max(3, min(args.steps, 10))
    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gpu_busy()
    e0.record(st)
    for _ in range(steps):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    t_ms = e0.elapsed_time(e1)
    if use_dist:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = tt.item()
    if fused:
        peers.sync()
        res = peers.local
    elif use_dist:
        res = glob
    else:
        res = ctr
    got = res.cpu().numpy().view(np.uint64)[:w]
    want = golden_total("c5_w16_64gib_total")
    k = warm + steps
    exact = None if want is None else bool(all(int(g) == k * x for g, x in zip(got, want)))
    if fused:
        peers.zero()
    del shard
    torch.cuda.empty_cache()
    gbs = total * steps / (t_ms / 1e3) / 1e9
    return {"value": round(gbs, 1), "unit": "GB/s", "ms_per_step": round(t_ms / steps, 4),
            "steps": steps, "warmup": warm, "n_gpus": world, "scaling": "strong",
            "bytes_total": total, "bytes_per_gpu": n,
            "exchange": ("fused in-kernel peer adds" if fused else
                         "NCCL allreduce per step" if use_dist else "none (one GPU)"),
            "hbm_frac_per_gpu": round(gbs / world / load_peaks()[0], 4),
            "exact": exact,
            "exact_reference": "steps x the reference numba total of the 64 GiB array "
                               "(tests/golden/golden.json c5_w16_64gib_total)"}


def main_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2412_16370_b200 as pp
    from paper_2412_16370_b200 import _lib, gen

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus is not None and args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one "
                         "rank per GPU (torchrun --nproc-per-node N, or plain --gpus N)")
    # PP_BENCH_DEVICE / PP_BENCH_BACKEND: test hooks that run N ranks on one
    # GPU over gloo (tests/test_gpu_bench_dist.py); never set for a measurement
    if "PP_BENCH_DEVICE" not in os.environ:
        require_devices(world, local)
    local = int(os.environ.get("PP_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    numa_cpus = bind_to_gpu_numa_node(local) if world > 1 else None
    dev = torch.device("cuda", local)
    # under torchrun (even with one rank) the NCCL path runs: every step ends
    # with the allreduce of the counters; plain `python bench.py` is N=1 local
    use_dist = "LOCAL_RANK" in os.environ or world > 1
    if use_dist and (args.exchange == "nccl" or args.config == "c3cat"):
        # leave 8 SMs to NCCL so each step's allreduce runs concurrently with
        # the next count (the count is HBM-bound: 140 SMs saturate it); the
        # fused exchange has no collective kernels and keeps every SM
        os.environ.setdefault("PP_RESERVE_SMS", "8")
    if use_dist:
        # NCCL's own log lines (e.g. "NCCL version ..." under NCCL_DEBUG) go to
        # stderr: stdout carries exactly one JSON line
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        backend = os.environ.get("PP_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    lib = _lib.load()
    st = torch.cuda.current_stream(dev)
    sp = st.cuda_stream

    cfg = args.config
    kind, w, nbytes, desc = CONFIGS[cfg]
    if args.width and cfg in ("c2",):
        w = args.width
    seed = {"c1": 0xC1, "c2": 0xC2, "c3": 0xC3, "c4": 0xC4, "c4seg": 0xC4 + 1, "c5": 0xC5,
            "c3cat": 0xC3}[cfg]
    categorical = cfg == "c3cat"
    offset = 3 if cfg == "c4" else 0
    word_unit = 4 if kind == "onehot32" else 8
    strong = cfg in STRONG
    if strong:
        # contiguous shard of the fixed-size array, cut at 64-byte multiples
        from paper_2412_16370_b200.dist import shard_range
        lo, hi = shard_range(nbytes, world, rank)
        nbytes = hi - lo
        alloc, first_word = nbytes, lo // word_unit
    else:
        alloc = nbytes + (64 if cfg == "c4" else 0)
        first_word = rank * alloc // word_unit
    buf = gen.generate(kind, alloc, seed, device=dev, word_offset=first_word, q=655)
    view_ptr = buf.data_ptr() + offset
    # R identical copies of the input in R slots of one buffer, step i
    # counting slot i mod R, steps back to back: every step's input was last
    # touched R - 1 steps (>= 510 MiB and >= 2 other inputs) earlier, so it
    # is cold in L2 without a flush between steps -- also when consecutive
    # launches overlap (the next count's loads start during this one,
    # INPUT_READY + the trigger at kernel start: two launches over ONE
    # buffer would share L2 lines).  C5 (one 64 GiB array) keeps one copy:
    # overlapping launches read it 64 GiB apart.  For inputs that fit in L2
    # (C1, C4) the flush-then-one-launch protocol is reported beside it as
    # the cold single-call latency.
    small = nbytes < L2_FLUSH_BELOW
    rot = None
    slot_ptrs = [view_ptr]
    if not strong and (cfg != "c4seg" or small):
        slot = (alloc + 4095) // 4096 * 4096  # keeps the view's address mod 4096
        nslot = max(3, -(-L2_FLUSH_BYTES // slot))
        rot = torch.empty(nslot * slot, dtype=torch.uint8, device=dev)
        rot.view(nslot, slot)[:, :alloc].copy_(buf.view(1, alloc).expand(nslot, alloc))
        slot_ptrs = [rot.data_ptr() + i * slot + offset for i in range(nslot)]
    torch.cuda.synchronize()

    # counters2[p] accumulates the steps of parity p.  Exchange pipeline: the
    # side stream snapshots counters2[i % 2] after step i's count and
    # allreduces the snapshot while the main stream counts step i+1 into the
    # other accumulator; the main stream only ever carries count kernels (plus
    # waits), and the timed region waits for every exchange (drain()).
    counters2 = torch.zeros((2, 64), dtype=torch.int64, device=dev)
    counters = counters2[0]
    # --exchange fused (default under torchrun for the plain count): no
    # collective per step; each rank's kernel adds every CTA's counts into all
    # ranks' IPC-mapped counters (pp_count_multi), so a step ends when the
    # kernel does and the max over ranks of the event timings covers it
    fused = use_dist and args.exchange == "fused" and not categorical and cfg != "c4seg"
    peers = None
    if fused:
        from paper_2412_16370_b200.dist import PeerCounters
        try:
            peers = PeerCounters(device=dev)
            ntgt = len(peers.targets)
        except RuntimeError as exc:  # no peer access between these GPUs: NCCL exchange
            print(f"bench: {exc}; using the NCCL exchange", file=sys.stderr)
            fused, peers = False, None
    globs = [torch.zeros(64, dtype=torch.int64, device=dev) for _ in range(2)]
    count_ev = [torch.cuda.Event() for _ in range(2)]
    snap_ev = [torch.cuda.Event() for _ in range(2)]
    red_ev = [torch.cuda.Event() for _ in range(2)]
    side = torch.cuda.Stream(dev) if use_dist else None
    nstep = [0]
    # the inputs are written once, before any count: each step's loads may
    # overlap the previous step's tail (pp_count_ex, PP_COUNT_INPUT_READY)
    count_flags = _lib.PP_COUNT_INPUT_READY if args.input_ready else 0
    seg_out = None
    if cfg == "c4seg":
        seg = 4096
        nseg = nbytes // seg
        seg_out = torch.zeros((nseg, w), dtype=torch.int64, device=dev)

    def step():
        b = nstep[0] % 2
        view_ptr = slot_ptrs[nstep[0] % len(slot_ptrs)]
        if seg_out is not None:
            _lib.check(lib.pp_count_fixed(view_ptr, 4096, nbytes // 4096, w, seg_out.data_ptr(),
                                          _lib.PP_SEG_OVERWRITE, sp))
        else:
            if fused:
                _lib.check(lib.pp_count_multi_ex(view_ptr, nbytes, w, peers.targets, ntgt,
                                                 count_flags, sp))
                nstep[0] += 1
                return
            if use_dist:
                st.wait_event(snap_ev[b])  # step i-2's snapshot of counters2[b] is taken
            if categorical:  # one u8 code per byte
                _lib.check(lib.pp_count_categories_ex(view_ptr, nbytes, 1, w,
                                                      counters2[b].data_ptr(), count_flags, sp))
            else:
                _lib.check(lib.pp_count_ex(view_ptr, nbytes, w, counters2[b].data_ptr(),
                                           count_flags, sp))
        if use_dist and seg_out is None:  # segmented rows stay on their rank
            count_ev[b].record(st)
            side.wait_event(count_ev[b])
            with torch.cuda.stream(side):
                side.wait_event(red_ev[b])  # globs[b] free again
                globs[b].copy_(counters2[b])
                snap_ev[b].record(side)
                dist.all_reduce(globs[b])
                red_ev[b].record(side)
        nstep[0] += 1

    def drain():
        if use_dist and not fused and seg_out is None:  # last exchanges inside the region
            st.wait_event(red_ev[0])
            st.wait_event(red_ev[1])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # settle: after the W warm-up steps, keep the GPU streaming the same
    # kernel over the same bytes (into scratch counters, so the exactness
    # checks below are untouched) for >= SETTLE_MS of device time: with only
    # W = 5 steps (0.7 ms) the first timed region occasionally ran 2-3 %
    # slow (7241 vs 7416-7444 GB/s on one box, scripts/gpu_warm.sh)
    scratch_s = torch.zeros(64, dtype=torch.int64, device=dev)
    if seg_out is not None:
        settle_one = lambda: _lib.check(lib.pp_count_fixed(  # noqa: E731
            view_ptr, 4096, nbytes // 4096, w, seg_out.data_ptr(), _lib.PP_SEG_OVERWRITE, sp))
    elif categorical:
        settle_one = lambda: _lib.check(lib.pp_count_categories(  # noqa: E731
            view_ptr, nbytes, 1, w, scratch_s.data_ptr(), sp))
    else:
        settle_one = lambda: _lib.check(lib.pp_count(  # noqa: E731
            view_ptr, nbytes, w, scratch_s.data_ptr(), sp))
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(st)
    settle_one()
    s1.record(st)
    torch.cuda.synchronize()
    n_settle = min(2000, int(SETTLE_MS / max(s0.elapsed_time(s1), 1e-3)) + 1)
    for _ in range(n_settle):
        settle_one()
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()

    # K back-to-back steps between one event pair; small inputs rotate over
    # their slots (above), larger ones stream past L2 by themselves
    nstep[0] = args.warmup  # timed steps start on slots the settle loop did not touch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.05)  # let the sampler start before the timed region
        clk.mark(True)
        gpu_busy()  # launches queue behind a spin, not an idle GPU
        e0.record(st)
        for _ in range(args.steps):
            step()
        drain()
        e1.record(st)
        torch.cuda.synchronize()
        clk.mark(False)
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_ms = e0.elapsed_time(e1)
    cold_call = None
    if small and not use_dist:
        # the other protocol for small inputs: flush L2 (write then read a
        # 512 MiB buffer), then one launch alone between its own events, into
        # scratch counters; per-call device latency of an isolated call
        flush_buf = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
        flush_sink = torch.zeros((), dtype=torch.int64, device=dev)
        times = []
        for _ in range(args.steps):
            flush_buf.fill_(1)
            flush_sink.copy_(flush_buf.view(torch.int64).max())
            a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_ev.record(st)
            settle_one()
            b_ev.record(st)
            times.append((a_ev, b_ev))
        torch.cuda.synchronize()
        us = [1e3 * a.elapsed_time(b) for a, b in times]
        cold_call = {"us_median": round(statistics.median(us), 2), "us_min": round(min(us), 2),
                     "gbs_median": round(nbytes / statistics.median(us) / 1e3, 1),
                     "calls": len(us),
                     "protocol": "L2 flushed (512 MiB written then read) before each call; one "
                                 "launch between its own CUDA events"}
        del flush_buf
    if not use_dist or fused:
        # each step is exactly one launch of the dominant kernel
        k_ms = t_ms / args.steps
    else:
        # kernel alone (no allreduce between launches), same stream, same clocks
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gpu_busy()  # launches queue behind a spin, not an idle GPU
        k0.record(st)
        scratch = torch.zeros(64, dtype=torch.int64, device=dev)
        for _ in range(args.steps):
            _lib.check(lib.pp_count(view_ptr, nbytes, w, scratch.data_ptr(), sp))
        k1.record(st)
        torch.cuda.synchronize()
        k_ms = k0.elapsed_time(k1) / args.steps
    if use_dist:
        tt = torch.tensor([t_ms, k_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms, k_ms = tt.tolist()
    per_step_bytes = nbytes  # this rank's bytes per step
    job_bytes = per_step_bytes
    if use_dist:
        jb = torch.tensor([per_step_bytes], dtype=torch.int64, device=dev)
        dist.all_reduce(jb)
        job_bytes = int(jb.item())
    value = job_bytes * args.steps / (t_ms / 1e3) / 1e9

    # exactness: C5 against the reference's own 64 GiB total (golden file),
    # the others against the CPU oracle on this rank's shard
    exact = None
    if args.check and cfg == "c5" and rank == 0:
        want = golden_total("c5_w16_64gib_total")
        src = peers.local if fused else (globs[0] + globs[1]) if use_dist else counters2.sum(0)
        got = src.cpu().numpy().view(np.uint64)[:w]
        total = args.warmup + args.steps
        exact = None if want is None else bool(
            all(int(g) == total * x for g, x in zip(got, want)))
    elif args.check and categorical and rank == 0 and not use_dist:
        # same draws as C3's one-hot words: the reference's own C3 counters
        with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
            want = {c["name"]: c for c in json.load(f)["cases"]}["c3_w32_onehot_4gib"]["numba"]
        got = counters2.sum(0).cpu().numpy().view(np.uint64)[:w]
        total = args.warmup + args.steps
        exact = bool(all(int(g) == total * x for g, x in zip(got, want)))
    elif args.check and fused and cfg in ("c1", "c2", "c3", "c4"):
        # every rank's oracle on its own shard, summed over ranks, against the
        # job total the fused exchange left in this rank's counters
        from oracle import oracle as O
        host = buf.cpu().numpy()
        want = torch.tensor(O.hs512(host, offset, nbytes, w,
                                    threads=max(1, host_threads() // world)),
                            dtype=torch.int64, device=dev)
        del host
        dist.all_reduce(want)
        total = args.warmup + args.steps
        ok = torch.tensor([int(bool(torch.equal(peers.local[:w], total * want)))],
                          dtype=torch.int64, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        exact = bool(ok.item())
    elif args.check and seg_out is not None:
        # every row of this rank's segments against the oracle's per-segment
        # count (rows were overwritten by each step: one pass)
        from oracle import oracle as O
        host = buf[:nbytes].cpu().numpy()
        offs = np.arange(nbytes // 4096 + 1, dtype=np.uint64) * 4096
        want = O.segments(host, offs, w, threads=max(1, host_threads() // world))
        exact = bool(np.array_equal(seg_out.cpu().numpy().view(np.uint64), want))
        if use_dist:
            ok = torch.tensor([int(exact)], dtype=torch.int64, device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            exact = bool(ok.item())
        del host
    elif args.check and cfg in ("c1", "c2", "c3", "c4") and rank == 0:
        from oracle import oracle as O
        host = buf.cpu().numpy()
        want = O.hs512(host, offset, nbytes, w, threads=host_threads())
        got = counters2.sum(0).cpu().numpy().view(np.uint64)[:w]
        total = args.warmup + args.steps
        exact = bool(all(int(g) == total * x for g, x in zip(got, want)))
        del host

    # the metric is per word width: the same resident bytes at every other w
    # (one launch per step, CUDA events around the steps, this rank's GB/s)
    per_width = None
    if seg_out is None and cfg == "c2":
        per_width = {}
        scratch_w = torch.zeros(64, dtype=torch.int64, device=dev)
        for ww in (8, 16, 32, 64):
            if nbytes % (ww // 8):
                continue
            ns = len(slot_ptrs)
            for i in range(2):
                _lib.check(lib.pp_count_ex(slot_ptrs[i % ns], nbytes, ww, scratch_w.data_ptr(),
                                           count_flags, sp))
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            gpu_busy()  # launches queue behind a spin, not an idle GPU
            q0.record(st)
            for i in range(args.steps):
                _lib.check(lib.pp_count_ex(slot_ptrs[(2 + i) % ns], nbytes, ww,
                                           scratch_w.data_ptr(), count_flags, sp))
            q1.record(st)
            torch.cuda.synchronize()
            per_width[str(ww)] = round(nbytes * args.steps / (q0.elapsed_time(q1) / 1e3) / 1e9, 1)

    # C4's short / unaligned sweep: device time per call for every length of
    # BASELINE config 4 at byte offsets 1..7 (latency-bound below ~16 MiB)
    c4_sweep = None
    if cfg == "c4":
        c4_sweep = {"_note": "per-call device latency, launches queued back to back over the "
                             "same buffer (L2 warm; the sizes below 1 MiB are launch-bound)"}
        scratch_c = torch.zeros(64, dtype=torch.int64, device=dev)
        for words in (1, 3, 17, 255, 512, 8192, 131072, 8388608):
            nb = 8 * words
            reps = 200 if nb <= (1 << 20) else 50
            for _ in range(5):
                _lib.check(lib.pp_count(buf.data_ptr() + 1, nb, 64, scratch_c.data_ptr(), sp))
            gpu_busy()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            q0.record(st)
            for r in range(reps):
                off = 1 + r % 7
                _lib.check(lib.pp_count(buf.data_ptr() + off, nb, 64, scratch_c.data_ptr(), sp))
            q1.record(st)
            torch.cuda.synchronize()
            us = q0.elapsed_time(q1) / reps * 1e3
            c4_sweep[str(words)] = {"us_per_call": round(us, 2),
                                    "GBs": round(nb / us / 1e3, 2)}
        # the same lengths batched: up to 1M arrays of each length (<= 64 MiB)
        # at byte offset 3, one pp_count_fixed launch, one counter row each
        out_b = torch.empty(((1 << 20) * 64,), dtype=torch.int64, device=dev)
        for words in (1, 3, 17, 255, 512, 8192):
            seg = 8 * words
            nseg = min(1 << 20, (nbytes - 8) // seg)
            fb = lambda: _lib.check(lib.pp_count_fixed(buf.data_ptr() + 3, seg, nseg, 64,
                                                       out_b.data_ptr(), _lib.PP_SEG_OVERWRITE, sp))
            for _ in range(3):
                fb()
            gpu_busy()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            q0.record(st)
            for _ in range(10):
                fb()
            q1.record(st)
            torch.cuda.synchronize()
            us = q0.elapsed_time(q1) / 10 * 1e3
            c4_sweep[f"{words}_batched"] = {"arrays": nseg, "us_per_launch": round(us, 2),
                                            "ns_per_array": round(us * 1e3 / nseg, 3),
                                            "in_plus_out_GBs": round((seg + 512) * nseg / us / 1e3, 1)}
        del out_b

    # the paper's read-only "roofline" kernel over the same bytes, launched
    # and rotated over the input copies exactly like the count steps
    # (starting half a rotation away from the copies the timed steps read)
    sink = torch.zeros(1, dtype=torch.int64, device=dev)
    nslots = len(slot_ptrs)
    s0 = args.warmup + args.steps + nslots // 2
    for i in range(max(3, args.warmup)):
        _lib.check(lib.pp_readonly_sum_ex(slot_ptrs[(s0 + i) % nslots], nbytes,
                                          sink.data_ptr(), count_flags, sp))
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nro = max(5, args.steps)
    gpu_busy()  # launches queue behind a spin, not an idle GPU
    r0.record(st)
    for i in range(nro):
        _lib.check(lib.pp_readonly_sum_ex(slot_ptrs[(s0 + max(3, args.warmup) + i) % nslots],
                                          nbytes, sink.data_ptr(), count_flags, sp))
    r1.record(st)
    torch.cuda.synchronize()
    ro_gbs = nbytes * nro / (r0.elapsed_time(r1) / 1e3) / 1e9

    peak, peak_src = load_peaks()
    achieved = per_step_bytes / (k_ms / 1e3) / 1e9
    seg_tma = os.environ.get("PP_SEG_PATH", "") != "ldg" and view_ptr % 16 == 0
    kernel_key = (("pp_segtma_kernel<8>" if seg_tma else "pp_seg_kernel") if seg_out is not None else
                  f"pp_tma_kernel<{w}, 16>" if categorical else "pp_tma_kernel<1>")
    traffic, traffic_ratio = load_traffic(kernel_key, per_step_bytes)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": kernel_key, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": per_step_bytes,
                "traffic_per_input_byte_ncu": traffic_ratio,
                "readonly_roofline_gbs": round(ro_gbs, 1),
                # B200 HBM3e datasheet figure (HGX; 8 TB/s DGX), stated as such
                "spec_peak_gbs": SPEC_HBM_GBS,
                "frac_of_spec": round(achieved / SPEC_HBM_GBS, 4)}
    if categorical:
        # the fused producer is ALU-bound, not HBM-bound (profiles/r2_cat_ncu.md):
        # ALU-pipe lane-ops per code (ncu, this build) x codes/s (live) against
        # 148 SMs x 64 lane-ops/clk x the SM clock sampled in the region
        alu, lds = load_alu(kernel_key)
        if alu is not None:
            mhz = clk.summary().get("sm_mhz") or 1965.0
            ops = alu * per_step_bytes / (k_ms / 1e3) / 1e12
            apeak = 148 * 64 * mhz * 1e6 / 1e12
            hbm = dict(roofline)
            roofline = {"bound": "alu", "achieved": round(ops, 3), "peak": round(apeak, 3),
                        "unit": "T lane-ops/s", "frac": round(ops / apeak, 4),
                        "traffic": traffic, "kernel": kernel_key,
                        "alu_lane_ops_per_code_ncu": alu,
                        # the second pipe the kernel leans on: shared-memory
                        # wavefronts (codes' LDS.U8 + table loads) against one
                        # wavefront per clock per SM
                        "smem_pipe_frac": (round(lds * per_step_bytes / (k_ms / 1e3)
                                                 / (148 * mhz * 1e6), 4) if lds else None),
                        "peak_source": f"148 SMs x 64 ALU-pipe lane-ops/clk x {mhz:.0f} MHz "
                                       "(median SM clock in the timed region)",
                        "hbm": {k: hbm[k] for k in ("achieved", "peak", "unit", "frac",
                                                    "readonly_roofline_gbs")}}
    if seg_out is not None:
        seg_bytes_out = (nbytes // 4096) * w * 8
        roofline["algorithmic_bytes_per_launch"] = per_step_bytes + seg_bytes_out
        roofline["achieved"] = round((per_step_bytes + seg_bytes_out) / (k_ms / 1e3) / 1e9, 1)
        roofline["frac"] = round(roofline["achieved"] / peak, 4)

    # e2e through the public API from pinned host memory
    e2e = None
    e2e_pageable = None
    if args.e2e and seg_out is None and nbytes <= 4 * GIB:
        pinned = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        pinned.copy_(buf[offset:offset + nbytes])
        torch.cuda.synchronize()
        nst = max(2, min(args.steps, 5))
        if use_dist and not categorical:
            # the job's public call at N ranks: every rank's host-resident
            # shard through its own link (pp_count_host), the w counters
            # all-reduced over the process group, the total read back
            from paper_2412_16370_b200.dist import pospopcnt_sharded
            api = lambda data, width: pospopcnt_sharded(data, width).cpu()  # noqa: E731
            e2e_path = ("pospopcnt_sharded(pinned host shard) on every rank: pp_count_host "
                        "(64 MiB chunks, H2D on a copy stream overlapped with counting), the "
                        "counters all-reduced over NCCL and read back")
        else:
            api = pp.pospopcnt_categories if categorical else pp.pospopcnt
            e2e_path = ("pospopcnt(pinned host tensor) -> pp_count_host: 64 MiB chunks, "
                        "H2D on a copy stream overlapped with counting")
        for _ in range(1):
            api(pinned, w)
        if use_dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(nst):
            res = api(pinned, w)  # H2D inside, D2H of the w counters
        t_e2e = time.perf_counter() - t0
        if use_dist:
            tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = tt.item()
        e2e = {"value": round(world * nbytes * nst / t_e2e / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": w * 8,
               "path": e2e_path, "steps": nst}
        if not use_dist and not categorical:
            # the same call on PAGEABLE host memory (what the reference's
            # callers pass: bytes / numpy arrays / a mapped file): staged
            # through pinned pieces by the library's copy pool
            pageable = pinned.numpy().copy()
            pp.pospopcnt(pageable, w)
            t0 = time.perf_counter()
            for _ in range(nst):
                res = pp.pospopcnt(pageable, w)
            e2e_pageable = {"value": round(nbytes * nst / (time.perf_counter() - t0) / 1e9, 3),
                            "unit": "GB/s", "steps": nst,
                            "path": "pospopcnt(numpy array in pageable memory) -> pp_count_host: "
                                    "<= 8 MiB pinned staging pieces filled by the host copy pool "
                                    "(non-temporal stores), H2D and counting pipelined behind it"}
            del pageable
        del pinned, res
    elif args.e2e and seg_out is not None:
        # segmented batch from host memory through the public API: the batch
        # is copied to the device in 64 MiB pieces on a copy stream while the
        # previous piece's segments are counted (pospopcnt_fixed on the
        # current stream), then the counter rows are read back
        pinned = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        pinned.copy_(buf[:nbytes])
        rows_host = torch.empty((nbytes // 4096, w), dtype=torch.int64, pin_memory=True)
        dev_in = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        rows_dev = torch.empty((nbytes // 4096, w), dtype=torch.int64, device=dev)
        cs, ds = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        piece = 64 * MIB

        def e2e_step():
            for p0 in range(0, nbytes, piece):
                p1 = min(nbytes, p0 + piece)
                r0, r1 = p0 // 4096, p1 // 4096
                with torch.cuda.stream(cs):
                    dev_in[p0:p1].copy_(pinned[p0:p1], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(cs)
                st.wait_event(ev)
                pp.pospopcnt_fixed(dev_in[p0:p1], 4096, w, out=rows_dev[r0:r1],
                                   accumulate=False)
                cev = torch.cuda.Event()
                cev.record(st)
                with torch.cuda.stream(ds):  # rows D2H overlaps the next piece's H2D
                    ds.wait_event(cev)
                    rows_host[r0:r1].copy_(rows_dev[r0:r1], non_blocking=True)
            ds.synchronize()

        e2e_step()
        nst = max(2, min(args.steps, 5))
        if use_dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(nst):
            e2e_step()
        t_e2e = time.perf_counter() - t0
        if use_dist:
            tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = tt.item()
        e2e = {"value": round(world * nbytes * nst / t_e2e / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": (nbytes // 4096) * w * 8,
               "path": "pinned host batch -> 64 MiB H2D pieces on a copy stream overlapped "
                       "with pospopcnt_fixed per piece, each piece's counter rows D2H on a "
                       "third stream (full-duplex link)",
               "steps": nst}
        del pinned, rows_host, dev_in, rows_dev

    # e2e fanned out over every visible GPU (one host link each) through the
    # same public call: pospopcnt(pinned host tensor, w, devices="all")
    e2e_fanout = None
    if args.e2e and world == 1 and seg_out is None and not categorical:
        ndev = torch.cuda.device_count()
        if ndev > 1:
            pinned = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
            pinned.copy_(buf[offset:offset + nbytes])
            devs = list(range(ndev))
            pp.pospopcnt(pinned, w, devices=devs)
            nst = max(2, min(args.steps, 5))
            t0 = time.perf_counter()
            for _ in range(nst):
                res = pp.pospopcnt(pinned, w, devices=devs)
            t_f = time.perf_counter() - t0
            e2e_fanout = {"value": round(nbytes * nst / t_f / 1e9, 3), "unit": "GB/s",
                          "devices": devs, "h2d_bytes_per_step": nbytes,
                          "d2h_bytes_per_step": w * 8 * ndev, "steps": nst,
                          "path": "pospopcnt(pinned host tensor, w, devices=all) -> "
                                  "pp_count_host_multi: one 64-byte-cut range per device, each "
                                  "through its own staging ring and host link"}
            del pinned, res
        else:
            e2e_fanout = {"skipped": "one GPU visible: the fan-out has a single link "
                                     "(tests/test_gpu_fanout.py covers its logic)"}

    cpu = None
    if args.cpu_baseline and world == 1 and rank == 0:
        sample = min(nbytes, 256 * MIB)
        cpu = cpu_leg(cfg, sample if cfg != "c4" else 64 * MIB, args.cpu_min_time)
        if cfg == "c4":
            cpu["sample"] += " (aligned; the GPU arm's view starts at byte offset 3)"

    # C5 strong scaling beside the weak-scaling headline: the fixed 64 GiB
    # array split over the N ranks, exact against the reference's own total
    strong_c5 = None
    if args.strong_c5 and cfg == "c2":
        del buf
        torch.cuda.empty_cache()
        strong_c5 = run_strong_c5(args, lib, world, rank, dev, st, use_dist, peers)

    # the other BASELINE configs as one summary each, measured in this run
    # (one child bench.py per config, after this config's own timing)
    others = None
    if args.all_configs and cfg == "c2" and not use_dist and args.width in (0, 8):
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        others = run_other_configs(args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": "u8" if w == 8 else f"u{w}",
            "data": "synthetic: seeded splitmix64 generators, generated in place in HBM",
            "config": config_dict(cfg, world, per_step_bytes, job_bytes, w),
            "launch": ("pp_count_ex(..., PP_COUNT_INPUT_READY): inputs written once before "
                       "the first count, so a step's loads may overlap the previous step's tail"
                       if count_flags and seg_out is None else "plain launches"),
            "host_binding": (f"each rank's host threads pinned to its GPU's NUMA-local CPUs "
                             f"(rank 0: {numa_cpus})" if numa_cpus else None),
            "exchange": ("none (rows stay on their rank)" if seg_out is not None else
                         "fused: the counting kernel adds into every rank's IPC-mapped "
                         "counters (pp_count_multi)" if fused else
                         f"NCCL allreduce of the {w} counters per step, pipelined on a side "
                         "stream") if world > 1 else "none (one GPU)",
            "timing": {"settle": f"{n_settle + 1} untimed launches (>= {SETTLE_MS:.0f} ms) "
                                 "after the warm-up steps, into scratch counters",
                       "l2": ("one input >> 126 MB L2, launches overlap 64 GiB apart"
                              if len(slot_ptrs) == 1 else
                              f"inputs larger than L2: {len(slot_ptrs)} copies of the input "
                              f"({len(slot_ptrs) * nbytes >> 20} MiB), step i counts copy "
                              f"i mod {len(slot_ptrs)}, steps back to back")},
            "cold_call": cold_call,
            "hbm_frac": round(value / world / peak, 4),
            "exact_reference": "C5: reference numba total of the 64 GiB array (golden.json)"
                               if cfg == "c5" else "CPU oracle (C port of NumbaKernel.run) "
                                                   + ("of every rank's shard, summed" if fused
                                                      else "on rank 0's shard"),
            "words_per_s": round(value * 1e9 / (w // 8)),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_pageable": e2e_pageable,
            "e2e_fanout": e2e_fanout,
            "strong_c5": strong_c5,
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "exact": exact,
            "per_width_gbs": per_width,
            "c4_short_sweep": c4_sweep,
            "other_configs": others,
        }
        emit(line)
    if peers is not None:
        peers.sync()
        peers.close()
    if use_dist:
        dist.destroy_process_group()
    return 0


OTHER_CONFIGS = ("c1", "c3", "c4", "c4seg", "c3cat")


def run_other_configs(args):
    """One child `bench.py --config X` per other BASELINE config (same GPU,
    same K/W, no e2e / CPU legs); returns {config: summary of its line}."""
    out = {}
    for cfg in OTHER_CONFIGS:
        cmd = [sys.executable, os.path.abspath(__file__), "--config", cfg,
               "--steps", str(args.steps), "--warmup", str(args.warmup), "--no-e2e",
               "--no-cpu-baseline", "--no-strong-c5", "--no-all-configs"]
        if not args.input_ready:
            cmd.append("--no-input-ready")
        t0 = time.time()
        try:
            res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
            lines = [x for x in res.stdout.splitlines() if x.strip().startswith("{")]
            if res.returncode != 0 or not lines:
                out[cfg] = {"error": f"rc={res.returncode}: {res.stderr.strip()[-300:]}"}
                continue
            d = json.loads(lines[-1])
        except Exception as exc:  # noqa: BLE001 - recorded, the headline stands
            out[cfg] = {"error": repr(exc)[:300]}
            continue
        r = d.get("roofline") or {}
        out[cfg] = {"workload": d["config"]["workload"], "value": d["value"], "unit": d["unit"],
                    "ms_per_step": d["ms_per_step"], "exact": d.get("exact"),
                    "roofline": {k: r.get(k) for k in ("bound", "achieved", "peak", "unit",
                                                       "frac", "kernel")},
                    "timing": d.get("timing"), "cold_call": d.get("cold_call"),
                    "launch": d.get("launch"), "clocks": d.get("clocks"),
                    "wall_s": round(time.time() - t0, 1)}
    return out


_JSON_OUT = None  # the real stdout: the one JSON line goes here, nothing else


def claim_stdout():
    """Point fd 1 at stderr for the rest of the run and keep a private copy
    of the real stdout for the JSON line: NCCL (e.g. NCCL_DEBUG=VERSION prints
    "NCCL version ..." on stdout at init), CUDA or torch messages must not
    mix into the one line the driver parses."""
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_torchrun(args):
    """`bench.py --gpus N` outside torchrun: one rank per GPU, as the driver
    launches it (python -m torch.distributed.run --nnodes=1 --nproc-per-node
    N --master-addr 127.0.0.1 ...).  The ranks' stdout is the real stdout
    (the one JSON line of rank 0)."""
    if "PP_BENCH_DEVICE" not in os.environ:
        require_devices(args.gpus)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    return subprocess.run(cmd, stdout=out, env=env).returncode


def main():
    claim_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="GPUs = ranks (default: WORLD_SIZE under torchrun, else 1); outside "
                         "torchrun N > 1 relaunches under torch.distributed.run")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--config", choices=tuple(CONFIGS), default="c2")
    ap.add_argument("--width", type=int, default=0, help="override w for c2 (sweep)")
    ap.add_argument("--exchange", choices=("fused", "nccl"), default="fused",
                    help="N>1 counter exchange: in-kernel remote adds, or NCCL allreduce")
    ap.add_argument("--no-check", dest="check", action="store_false")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--cpu-min-time", type=float, default=5.0)
    ap.add_argument("--no-input-ready", dest="input_ready", action="store_false",
                    help="count with plain pp_count (loads wait for the previous kernel)")
    ap.add_argument("--no-all-configs", dest="all_configs", action="store_false",
                    help="skip the other BASELINE configs' summaries in the c2 line")
    ap.add_argument("--no-strong-c5", dest="strong_c5", action="store_false",
                    help="skip the C5 strong-scaling object of the c2 line")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus is not None and args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if args.gpus and args.gpus > 1 and "LOCAL_RANK" not in os.environ:
        return relaunch_torchrun(args)
    return main_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
