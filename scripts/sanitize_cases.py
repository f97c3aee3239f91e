#!/usr/bin/env python3
"""Edge-case driver for `compute-sanitizer --tool memcheck` (and racecheck).

Run with PYTORCH_NO_CUDA_MEMORY_CACHING=1 so every tensor is its own
cudaMalloc of exactly the requested size: a read one byte past a view that
ends at its allocation's end is then reported.  Views start at every offset
0..15 of an allocation that holds exactly offset + n bytes; segmented batches
cover ragged/misaligned/empty segments ending at the allocation end.
Checks results against the CPU oracle too (test infrastructure).
"""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import paper_2412_16370_b200 as pp
    from oracle import oracle as O
    assert os.environ.get("PYTORCH_NO_CUDA_MEMORY_CACHING") == "1"
    rng = random.Random(5)
    checked = 0
    for w in (8, 16, 32, 64):
        step = w // 8
        for n in (0, step, 8, 15 * step, 16, 24, 40, 100 * step, 4096, 32768 + 40, 70000):
            n -= n % step
            for off in range(16):
                host = np.frombuffer(rng.randbytes(off + n), np.uint8)
                buf = torch.from_numpy(host.copy()).cuda()  # exactly off + n bytes
                c = torch.zeros(w, dtype=torch.int64, device="cuda")
                pp.pospopcnt(pp.InputView(buf, off, n), w, counters=c)
                assert [int(x) for x in c.cpu()] == O.hs512(host, off, n, w), (w, n, off)
                checked += 1
                del buf
    # segmented: ragged, misaligned, empty segments; last one ends at the allocation end
    for w in (8, 64):
        step = w // 8
        for lanes in (1, 8, 16, 32):
            lens = [rng.choice((0, step, 3 * step, 17 * step, 4096, 5000 - 5000 % step))
                    for _ in range(300)]
            offs = np.zeros(len(lens) + 1, dtype=np.int64)
            offs[1:] = np.cumsum(lens)
            base = 3
            host = np.frombuffer(rng.randbytes(int(offs[-1]) + base), np.uint8)
            buf = torch.from_numpy(host.copy()).cuda()
            out = pp.pospopcnt_segmented(pp.InputView(buf, base, int(offs[-1])), offs, w,
                                         lanes=lanes)
            want = O.segments(host, (offs + base).astype(np.uint64), w)
            assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (w, lanes)
            checked += 1
    # fixed segments (one lane per array below 1 KiB) ending at the allocation end
    for seg, w in ((8, 64), (24, 8), (136, 16), (4096, 32)):
        for off in (0, 5):
            nseg = 777
            host = np.frombuffer(rng.randbytes(off + nseg * seg), np.uint8)
            buf = torch.from_numpy(host.copy()).cuda()
            out = pp.pospopcnt_fixed(pp.InputView(buf, off, nseg * seg), seg, w)
            want = O.segments(host, (np.arange(nseg + 1, dtype=np.uint64) * seg + off), w)
            assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (seg, w, off)
            checked += 1
            del buf
    # one pass for all widths, host path
    host = np.frombuffer(rng.randbytes(4099), np.uint8)
    buf = torch.from_numpy(host.copy()).cuda()
    got = pp.pospopcnt_all_widths(pp.InputView(buf, 3, 4096))
    assert got[64] == O.hs512(host, 3, 4096, 64)
    assert pp.pospopcnt(host[1:4097].tobytes(), 32) == O.hs512(host, 1, 4096, 32)
    torch.cuda.synchronize()
    print(f"sanitize cases ok: {checked} views / batches")


if __name__ == "__main__":
    main()
