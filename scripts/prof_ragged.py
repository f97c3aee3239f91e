#!/usr/bin/env python3
"""ncu driver: the LDG-fed segmented kernel on 1 GiB of ragged 0-8 KiB CSR
segments (two launches; A/B of the load cache hint via PP_LIB_PATH)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2412_16370_b200 import _lib, gen
lib = _lib.load()
n = 1 << 30
buf = gen.generate("bernoulli", n + 64, 0xC5, q=655)
lens = np.random.default_rng(1).integers(0, 1024, 200_000) * 8
offs = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)])).cuda()
out = torch.empty((lens.size, 64), dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    _lib.check(lib.pp_count_segmented(buf.data_ptr(), offs.data_ptr(), lens.size, 64,
                                      out.data_ptr(), 1, sp))
torch.cuda.synchronize()
print("ok")
