#!/usr/bin/env python3
"""A few small synchronous calls for a launch list: host bytes -> list and
device view -> list at 4 KiB, 32 KiB + 16, 256 KiB and 4 MiB (device), each
call one kernel launch on the direct path (PP_NO_DIRECT=1: memset + count +
D2H copy instead).

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/direct_launches.csv python scripts/direct_calls.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_16370_b200 as pp  # noqa: E402

buf = torch.randint(0, 256, (4 << 20,), dtype=torch.uint8, device="cuda")
host = buf.cpu().numpy().tobytes()
torch.cuda.synchronize()
for n in (4096, 32768 + 16, 262144):
    a = pp.pospopcnt(host[:n], 16)
    b = pp.pospopcnt(pp.InputView(buf, 0, n), 16)
    assert a == b, n
print(sum(pp.pospopcnt(buf, 16)))
