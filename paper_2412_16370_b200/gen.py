"""Seeded synthetic inputs generated in place on the GPU (bench/test infrastructure).

Definitions in csrc/pp_gen.cu; byte-identical CPU twins in
oracle/pospopcnt_oracle.c.  BASELINE.json names no public dataset: these
stand in for the configs' distributions:

  uniform     C1/C2: i.i.d. Bernoulli(0.5) bits
  bernoulli   C4: i.i.d. Bernoulli(q/65536) bits (q=655 -> p=0.009995)
  blocks      C5: Bernoulli(q_b/65536) with q_b uniform on [0, 65536] per block
  onehot32    C3: u32 words with one set bit, bounded Zipf(1.1) over 32 positions
  codes8      C3 as u8 category codes (code i = bit position of onehot32 word i)
"""

import numpy as np
import torch

from . import _lib

SEEDS = {"c1": 0xC1, "c2": 0xC2, "c3": 0xC3, "c4": 0xC4, "c5": 0xC5}


def zipf_thresholds(s=1.1, k=32):
    """thr[i] = round(2^32 * P(cat <= i)) for a bounded Zipf(s) on {1..k}."""
    pmf = np.array([(i + 1) ** -s for i in range(k)], dtype=np.float64)
    pmf /= pmf.sum()
    cdf = np.cumsum(pmf)[:-1]
    return np.minimum(np.round(cdf * 2.0 ** 32), 2.0 ** 32 - 1).astype(np.uint32)


def generate(kind, nbytes, seed, device="cuda", word_offset=0, q=655,
             block_bytes=1 << 20, out=None):
    """A CUDA uint8 tensor of nbytes generated in place (asynchronous)."""
    lib = _lib.load()
    dev = torch.device(device)
    if out is None:
        out = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    dev = out.device
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev).cuda_stream
        ptr = out.data_ptr()
        if kind == "uniform":
            rc = lib.pp_gen_uniform(ptr, nbytes, seed, word_offset, st)
        elif kind == "bernoulli":
            rc = lib.pp_gen_bernoulli(ptr, nbytes, seed, word_offset, q, st)
        elif kind == "blocks":
            rc = lib.pp_gen_blocks(ptr, nbytes, seed, word_offset, block_bytes, st)
        elif kind == "onehot32":
            thr = zipf_thresholds()
            rc = lib.pp_gen_onehot32(ptr, nbytes, seed, word_offset, thr.ctypes.data, st)
        elif kind == "codes8":  # one u8 code per byte; one_hot(code i) == onehot32 word i
            thr = zipf_thresholds()
            rc = lib.pp_gen_codes8(ptr, nbytes, seed, word_offset, thr.ctypes.data, st)
        else:
            raise ValueError(f"unknown generator {kind!r}")
    _lib.check(rc)
    return out
