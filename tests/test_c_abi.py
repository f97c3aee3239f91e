"""The C ABI from plain C (tests/c/abi_host_test.c), no Python in the loop.

Compiles the test program with gcc against include/pospopcnt_b200.h and the
in-tree libpospopcnt_b200.so (plus the oracle library as the checker) and
runs it: on a CPU-only host every compute call must report PP_ENODEV (no CPU
fallback); on a B200 pp_count_host must match the oracle over lengths, host
alignments, widths and concurrent threads.
"""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2412_16370_b200")


def _gpu_present():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


@pytest.fixture(scope="module")
def abi_binary(tmp_path_factory, oracle):
    from paper_2412_16370_b200 import build
    build.build()
    exe = str(tmp_path_factory.mktemp("cabi") / "abi_host_test")
    odir = os.path.join(ROOT, "oracle")
    cmd = ["gcc", "-O2", "-Wall", "-Wextra", "-Werror", "-std=c11", "-D_GNU_SOURCE",
           "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "c", "abi_host_test.c"),
           "-L", PKG, "-lpospopcnt_b200", "-L", odir, "-loracle",
           f"-Wl,-rpath,{PKG}:{odir}", "-pthread", "-o", exe]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return exe


@pytest.mark.skipif(_gpu_present(), reason="checks the no-GPU behaviour")
def test_c_abi_without_gpu_fails_loudly(abi_binary):
    res = subprocess.run([abi_binary, "--nodev"], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0 and res.stdout.strip() == "ok", res.stdout + res.stderr


@pytest.mark.gpu
def test_c_abi_host_path_matches_oracle(abi_binary):
    res = subprocess.run([abi_binary], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0 and res.stdout.strip() == "ok", res.stdout + res.stderr
