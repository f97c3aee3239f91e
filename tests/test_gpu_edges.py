"""Edge cases at exact allocation boundaries (scripts/sanitize_cases.py).

compute-sanitizer is closed on this GPU pool, so the memory-safety evidence is
by construction (exact-bounds byte loads for every partial vector) plus this
driver: every tensor is its own cudaMalloc of exactly offset + n bytes
(PYTORCH_NO_CUDA_MEMORY_CACHING=1), views end at the allocation end, and all
results must equal the CPU oracle.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exact_allocation_edges(cuda):
    env = dict(os.environ, PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_cases.py")],
                         env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert "sanitize cases ok" in res.stdout
