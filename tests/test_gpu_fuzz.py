"""A short run of the randomised differential soak (scripts/fuzz.py): random
entry points, sizes, offsets and widths from several host threads and
streams at once, each result against the oracle."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fuzz_short(cuda):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "fuzz.py"),
                          "--seconds", "30", "--threads", "3", "--seed", "7"],
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "failures: []" in res.stdout
