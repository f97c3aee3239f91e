#!/usr/bin/env python3
"""Small driver for ncu: launches each hot kernel a few times on C2/C4-sized
inputs (1 GiB), so `ncu -k regex:...` can capture them.

  python scripts/prof_kernels.py [--reps N] [--which count,readonly,seg]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--which", default="count,readonly,seg,cat")
    ap.add_argument("--width", type=int, default=8)
    args = ap.parse_args()
    import torch

    from paper_2412_16370_b200 import _lib, gen
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    sp = torch.cuda.current_stream().cuda_stream
    n = 1 << 30
    buf = gen.generate("uniform", n, 0xC2, device=dev)
    seg_buf = gen.generate("bernoulli", n, 0xC4 + 1, device=dev, q=655)
    cnt = torch.zeros(64, dtype=torch.int64, device=dev)
    sink = torch.zeros(1, dtype=torch.int64, device=dev)
    out = torch.zeros((n // 4096, 64), dtype=torch.int64, device=dev)
    which = args.which.split(",")
    codes = gen.generate("codes8", n, 0xC3, device=dev) if "cat" in which else None
    for _ in range(args.reps):
        if "count" in which:
            _lib.check(lib.pp_count(buf.data_ptr(), n, args.width, cnt.data_ptr(), sp))
        if "readonly" in which:
            _lib.check(lib.pp_readonly_sum(buf.data_ptr(), n, sink.data_ptr(), sp))
        if "seg" in which:
            _lib.check(lib.pp_count_fixed(seg_buf.data_ptr(), 4096, n // 4096, 64,
                                          out.data_ptr(), _lib.PP_SEG_OVERWRITE, sp))
        if "cat" in which:  # fused one-hot producer at every width (u8 codes)
            for w in (8, 16, 32, 64):
                _lib.check(lib.pp_count_categories(codes.data_ptr(), n, 1, w, cnt.data_ptr(), sp))
    torch.cuda.synchronize()
    print("ok", [int(x) for x in cnt[:args.width].cpu()][:4])


if __name__ == "__main__":
    main()
