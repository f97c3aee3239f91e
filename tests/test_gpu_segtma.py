"""Fixed-size segments through the TMA-ring kernel (pp_segtma_kernel) vs the oracle.

The dispatch (PP_SEG_PATH, read once per process) is forced to the TMA ring
in a child process so that small batches, partial last chunks, every lane
count and every width reach it; the same cases forced to the LDG kernel
must agree.  Row s must equal the reference's count of segment s alone
(NumbaKernel.run on InputView(base, s*seg, seg), kernels.py:242-270).
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from oracle import oracle as O
import paper_2412_16370_b200 as pp
from paper_2412_16370_b200 import gen
O.build()
cases = [
    # (seg_bytes, nseg, width, lanes)
    (4096, 1, 64, 8), (4096, 5, 64, 8), (4096, 4 * 148 * 16 + 7, 64, 8),
    (4096, 3000, 8, 32), (4096, 3001, 16, 16),
    (16, 10000, 8, 8), (48, 7777, 16, 8), (64, 4099, 64, 8), (1008, 999, 32, 8),
    (8192, 777, 64, 16), (8192, 333, 8, 8), (16384, 300, 32, 32), (16384, 65, 64, 32),
    (2064, 1234, 16, 16), (16400, 40, 8, 32),  # > one item per stage: LDG kernel
]
for seg, nseg, w, lanes in cases:
    buf = gen.generate("uniform", (nseg * seg + 7) // 8 * 8, seed=seg * 131 + nseg)
    host = buf.cpu().numpy()
    offs = np.arange(nseg + 1, dtype=np.uint64) * seg
    want = O.segments(host, offs, w)
    out = pp.pospopcnt_fixed(buf[:nseg * seg], seg, w, lanes=lanes)
    got = out.cpu().numpy().view(np.uint64)
    assert np.array_equal(got, want), (seg, nseg, w, lanes)
    # accumulate into the same rows, then overwrite
    pp.pospopcnt_fixed(buf[:nseg * seg], seg, w, out=out, lanes=lanes)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), 2 * want), (seg, nseg, w)
    pp.pospopcnt_fixed(buf[:nseg * seg], seg, w, out=out, accumulate=False, lanes=lanes)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (seg, nseg, w)
# a trailing partial segment is ignored; an unaligned base takes the LDG kernel
buf = gen.generate("uniform", 1 << 20, seed=7)
host = buf.cpu().numpy()
for off in (0, 3):
    v = buf[off:off + 4096 * 200 + 100]
    want = O.segments(host[off:off + 4096 * 200], np.arange(201, dtype=np.uint64) * 4096, 16)
    got = pp.pospopcnt_fixed(v, 4096, 16).cpu().numpy().view(np.uint64)
    assert np.array_equal(got, want), off
print("ok")
"""


@pytest.mark.parametrize("path", ("tma", "ldg"))
def test_fixed_segments_forced_path(cuda, path):
    env = dict(os.environ, PP_SEG_PATH=path)
    res = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0 and res.stdout.strip().endswith("ok"), res.stdout + res.stderr
