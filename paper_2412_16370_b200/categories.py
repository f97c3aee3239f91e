"""GROUP BY COUNT over categorical codes: the fused one-hot producer.

The paper's motivating use is the histogram of one-hot
encoded categories, i.e. ``pospopcnt`` over words ``1 << code``.  This entry
point takes the codes themselves and returns exactly

    pospopcnt_categories(codes, w)[j] == pospopcnt(one_hot_w(codes), w)[j]
                                      == #{i : codes[i] == j}

without materialising the w/8-byte one-hot words (codes >= w have no bit in a
w-bit word and are not counted; negative 2-/4-byte codes neither).  Computed
by pp_count_categories: the codes (1, 2 or 4 bytes each) are expanded into
packed one-hot words in registers on the TMA pipeline and counted by the
same carry-save counter as pospopcnt (csrc/pp_count.cu; the shared-memory
histogram of csrc/pp_categories.cu remains as the A/B alternative).
"""

import numpy as np

from . import _lib
from .core import KernelUnavailableError, check_width, is_torch_tensor, new_counters
from .kernels import _add_into, _device_counters, _device_scratch

_CODE_BYTES = {1: 1, 2: 2, 4: 4}


def pospopcnt_categories(codes, width, counters=None, *, input_ready=False):
    """Add the per-category counts of ``codes`` (< width) into ``counters``.

    ``codes``: a 1-D CUDA tensor of uint8 / int16 / uint16 / int32 / uint32
    codes (host arrays are copied to the current device once).  Counters
    follow the ``pospopcnt`` conventions: a CUDA int64 tensor is accumulated
    asynchronously on the device, anything else receives Python ints.
    ``input_ready``: as ``pospopcnt`` (the kernel queued before this count
    does not write the codes; pp_count_categories_ex, PP_COUNT_INPUT_READY).
    """
    import torch
    check_width(width)
    if not torch.cuda.is_available():
        raise KernelUnavailableError("pospopcnt_categories needs an sm_100 GPU (no CPU fallback)")
    if not is_torch_tensor(codes):
        codes = torch.as_tensor(np.ascontiguousarray(codes)).cuda()
    elif not codes.is_cuda:
        codes = codes.cuda()
    if codes.dim() != 1 or not codes.is_contiguous():
        raise ValueError("codes must be a contiguous 1-D tensor")
    cb = _CODE_BYTES.get(codes.element_size())
    if cb is None or codes.is_floating_point() or codes.dtype == torch.bool:
        raise ValueError("codes must be 1-, 2- or 4-byte integers")
    if counters is None:
        counters = new_counters(width)
    elif len(counters) < width:
        raise ValueError(f"counter array holds {len(counters)} < {width} entries")
    lib = _lib.load()
    n = codes.numel()
    if n == 0:
        return counters
    dev = codes.device
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        dc = _device_counters(counters, width, dev)
        if dc is not None:
            flags = _lib.PP_COUNT_INPUT_READY if input_ready else 0
            _lib.check(lib.pp_count_categories_ex(codes.data_ptr(), n, cb, width, dc.data_ptr(),
                                                  flags, stream))
            return counters
        scratch = _device_scratch(dev)
        scratch.zero_()
        _lib.check(lib.pp_count_categories(codes.data_ptr(), n, cb, width, scratch.data_ptr(),
                                           stream))
        vals = scratch[:width].cpu().numpy().view(np.uint64)
    _add_into(counters, vals, width)
    return counters
