#!/usr/bin/env python3
"""Randomised differential soak of the CUDA path against the CPU oracle.

Random sizes (0 .. ~300 MiB, so both chunk orders), offsets, widths, entry
points (device counts, host bytes, list / device counters, segmented, fixed,
batches of separate arrays, categories, all widths), several streams and host threads at once -- every
result checked against the oracle.  Runs for --seconds; exits 1 on the first
mismatch and prints the case.

  python scripts/fuzz.py --seconds 600 --threads 3
"""
import argparse
import os
import random
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_16370_b200 as pp  # noqa: E402
from oracle import oracle as O  # noqa: E402

MIB = 1 << 20


def one_case(rng, dev_buf, host, stream):
    kind = rng.choice(["count", "count", "count_list", "host", "seg", "fixed", "cat", "allw",
                       "batch"])
    w = rng.choice((8, 16, 32, 64))
    step = w // 8
    big = rng.random() < 0.15
    n = rng.randrange(0, (300 * MIB) if big else (4 * MIB)) // step * step
    off = rng.randrange(0, 64)
    n = min(n, host.size - off) // step * step
    with torch.cuda.stream(stream):
        if kind in ("count", "count_list", "host"):
            want = O.hs512(host, off, n, w, threads=4)
            if kind == "count":
                c = torch.zeros(w, dtype=torch.int64, device="cuda")
                # the buffer is written once before any count: input_ready
                # (pp_count_ex) is a valid promise here, half of the time
                pp.pospopcnt(pp.InputView(dev_buf, off, n), w, counters=c,
                             input_ready=rng.random() < 0.5)
                got = [int(x) for x in c.cpu()]
            elif kind == "count_list":
                got = pp.pospopcnt(pp.InputView(dev_buf, off, n), w)
            else:
                got = pp.pospopcnt(host[off:off + min(n, 8 * MIB) // step * step].tobytes(), w)
                want = O.hs512(host, off, min(n, 8 * MIB) // step * step, w, threads=4)
            return kind, (w, n, off), got == want
        if kind == "seg":
            if rng.random() < 0.9:
                nseg = rng.randrange(1, 3000)
                lens = [rng.choice((0, step, 7 * step, rng.randrange(0, 5000) // step * step,
                                    rng.randrange(0, 70000) // step * step)) for _ in range(nseg)]
            else:  # enough groups for scheduler batches of T > 1
                nseg = rng.randrange(50_000, 120_000)
                lens = (np.random.default_rng(rng.randrange(1 << 30)).integers(0, 4096 // step, nseg)
                        * step).tolist()
            offs = np.zeros(nseg + 1, dtype=np.int64)
            offs[1:] = np.cumsum(lens)
            if offs[-1] + off > host.size:
                return kind, "skip", True
            lanes = rng.choice((None, None, 1, 8, 16, 32))
            hybrid = rng.choice((None, False, True))
            view = pp.InputView(dev_buf, off, int(offs[-1]))
            if rng.random() < 0.3:  # a SegmentPlan (length-sorted order)
                plan = pp.SegmentPlan(offs, device="cuda", lanes=lanes, hybrid=hybrid)
                out = pp.pospopcnt_segmented(view, None, w, plan=plan)
                lanes = ("plan", plan.lanes)
            else:
                out = pp.pospopcnt_segmented(view, offs, w, lanes=lanes, hybrid=hybrid)
            want = O.segments(host, (offs + off).astype(np.uint64), w, threads=4)
            return kind, (w, nseg, off, lanes, hybrid), np.array_equal(
                out.cpu().numpy().view(np.uint64), want)
        if kind == "fixed":
            seg = rng.choice((8, 24, 256, 1024, 2048, 4096, 8192, 16384)) // step * step or step
            nseg = rng.randrange(1, (64 * MIB) // seg)
            if nseg * seg + off > host.size:
                return kind, "skip", True
            lanes = rng.choice((None, None, 1, 4, 8, 32))
            out = pp.pospopcnt_fixed(pp.InputView(dev_buf, off, nseg * seg), seg, w, lanes=lanes)
            want = O.segments(host, np.arange(nseg + 1, dtype=np.uint64) * seg + off, w,
                              threads=4)
            return kind, (w, seg, nseg, off, lanes), np.array_equal(
                out.cpu().numpy().view(np.uint64), want)
        if kind == "batch":
            k = rng.randrange(1, 400)
            spans = []
            for _ in range(k):
                ln = rng.choice((0, step, 9 * step, rng.randrange(0, 40000) // step * step))
                st = rng.randrange(0, host.size - ln + 1)
                spans.append((st, ln))
            lanes = rng.choice((None, None, 1, 8, 32))
            out = pp.pospopcnt_batch([pp.InputView(dev_buf, st, ln) for st, ln in spans], w,
                                     lanes=lanes)
            got = out.cpu().numpy().view(np.uint64)
            ok = all(list(got[i]) == O.hs512(host, st, ln, w) for i, (st, ln) in enumerate(spans))
            return kind, (w, k, lanes), ok
        if kind == "cat":
            dt = rng.choice((np.uint8, np.int16, np.int32))
            nc = rng.randrange(0, 2 * MIB)
            codes = np.random.default_rng(rng.randrange(1 << 30)).integers(
                -5 if dt != np.uint8 else 0, 100, nc).astype(dt)
            got = pp.pospopcnt_categories(torch.from_numpy(codes).cuda(), w)
            return kind, (w, nc, np.dtype(dt).name), got == O.categories(codes, w)
        # all widths from one pass
        got = pp.pospopcnt_all_widths(pp.InputView(dev_buf, off, n))
        ok = all(v == O.hs512(host, off, n, ww, threads=4) for ww, v in got.items())
        return kind, (n, off), ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=120)
    ap.add_argument("--threads", type=int, default=3)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    O.build()
    total = 320 * MIB
    host = np.random.default_rng(args.seed).integers(0, 256, total, dtype=np.uint8)
    dev = torch.from_numpy(host).cuda()
    torch.cuda.synchronize()
    stop = time.time() + args.seconds
    counts, failures, lock = {}, [], threading.Lock()

    def worker(i):
        rng = random.Random(args.seed * 1000 + i)
        stream = torch.cuda.Stream()
        while time.time() < stop and not failures:
            try:
                kind, case, ok = one_case(rng, dev, host, stream)
            except Exception as exc:  # noqa: BLE001
                kind, case, ok = "exception", repr(exc), False
            with lock:
                counts[kind] = counts.get(kind, 0) + 1
                if not ok:
                    failures.append((kind, case))

    ths = [threading.Thread(target=worker, args=(i,)) for i in range(args.threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    print("cases:", dict(sorted(counts.items())), "failures:", failures[:5], flush=True)
    return 1 if failures else 0


if __name__ == "__main__":
    sys.exit(main())
