import os
import random
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# the oracle is test infrastructure: tests may import it, the product never does
from oracle import oracle as O  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU")
    config.addinivalue_line("markers", "slow: long-running case")


def oracle_bits(data, w, counters=None):
    """Second scalar coding via bit strings (pkg/tests/conftest.py:9-19 idea)."""
    counters = counters if counters is not None else [0] * w
    data = bytes(data)
    step = w // 8
    for k in range(0, len(data), step):
        word = int.from_bytes(data[k:k + step], "little")
        for j, ch in enumerate(bin(word)[2:][::-1]):
            if ch == "1":
                counters[j] += 1
    return counters


@pytest.fixture
def rng():
    return random.Random(0xC0FFEE)


@pytest.fixture(scope="session")
def oracle():
    O.build()
    return O


@pytest.fixture(scope="session")
def cuda():
    """torch + the built library + an sm_100 device, or fail loudly (gpu tests)."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    import paper_2412_16370_b200 as pp
    from paper_2412_16370_b200 import _lib
    _lib.load()
    info = _lib.device_info(0)
    assert info["cc"][0] == 10, f"expected an sm_100 device, got {info}"
    return torch, pp
