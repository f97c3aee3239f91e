"""count FILE / stdin on the B200 (the reference's CLI count tests,
pkg/tests/test_cli.py:18-47, plus a file larger than the staging ring)."""

import io
import random

import numpy as np
import pytest

from paper_2412_16370_b200 import cli

pytestmark = pytest.mark.gpu


def run(capsys, *argv):
    code = cli.main(list(argv))
    out, err = capsys.readouterr()
    return code, out, err


def test_count_all_ones_file(cuda, tmp_path, capsys):
    f = tmp_path / "ff.bin"
    f.write_bytes(b"\xff\xff")
    code, out, _ = run(capsys, "count", "--width", "16", str(f))
    assert code == 0 and out.split() == ["1"] * 16


def test_count_empty_stdin_and_file(cuda, tmp_path, capsys, monkeypatch):
    monkeypatch.setattr("sys.stdin", io.TextIOWrapper(io.BytesIO(b"")))
    code, out, _ = run(capsys, "count", "--width", "8")
    assert code == 0 and out.split() == ["0"] * 8
    f = tmp_path / "empty.bin"
    f.write_bytes(b"")
    code, out, _ = run(capsys, "count", "--width", "64", str(f))
    assert code == 0 and out.split() == ["0"] * 64


def test_count_matches_oracle_and_csv(cuda, oracle, tmp_path, capsys):
    data = random.Random(5).randbytes(4096)
    f = tmp_path / "r.bin"
    f.write_bytes(data)
    code, out, _ = run(capsys, "count", "--width", "32", str(f))
    host = np.frombuffer(data, np.uint8)
    assert code == 0 and [int(v) for v in out.split()] == oracle.hs512(host, 0, 4096, 32)
    g = tmp_path / "x.bin"
    g.write_bytes(b"\x0f")
    code, out, _ = run(capsys, "count", "--width", "8", "--format", "csv", str(g))
    assert code == 0 and out.strip() == "1,1,1,1,0,0,0,0"


def test_count_large_file_memory_mapped(cuda, oracle, tmp_path, capsys):
    """96 MiB + 40 bytes: the mapped pages go through the pinned staging ring."""
    host = np.random.default_rng(3).integers(0, 256, (96 << 20) + 40, dtype=np.uint8)
    f = tmp_path / "big.bin"
    host.tofile(f)
    code, out, _ = run(capsys, "count", "--width", "64", str(f))
    assert code == 0
    assert [int(v) for v in out.split()] == oracle.hs512(host, 0, host.size, 64, threads=8)
