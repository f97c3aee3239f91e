"""The count / kernels command line (the reference's CLI tests,
pkg/tests/test_cli.py:18-75, for the paths that need no GPU here; the
counting cases run in tests/test_gpu_cli.py)."""

import pytest

from paper_2412_16370_b200 import cli


def run(capsys, *argv):
    code = cli.main(list(argv))
    out, err = capsys.readouterr()
    return code, out, err


def test_count_incomplete_input_exits_2(tmp_path, capsys):
    """pkg/tests/test_cli.py:50-55: validation precedes any device work."""
    f = tmp_path / "odd.bin"
    f.write_bytes(b"\x01\x02\x03")
    code, _, err = run(capsys, "count", "--width", "16", str(f))
    assert code == 2 and "multiple" in err


def test_count_missing_file_exits_2(capsys):
    code, _, _ = run(capsys, "count", "/no/such/file")
    assert code == 2


def test_count_unknown_kernel_exits_2(tmp_path, capsys):
    f = tmp_path / "x.bin"
    f.write_bytes(b"\x00")
    code, _, _ = run(capsys, "count", "--kernel", "warp9", str(f))
    assert code == 2


def test_bad_width_is_a_usage_error(capsys):
    with pytest.raises(SystemExit) as e:
        cli.main(["count", "--width", "12"])
    assert e.value.code == 2


def test_kernels_listing(capsys):
    code, out, _ = run(capsys, "kernels")
    assert code == 0
    lines = out.strip().splitlines()
    assert lines[0].startswith("b200")
    assert all(("available" in ln or "unavailable" in ln) for ln in lines)


def test_count_without_gpu_is_an_input_error(capsys, monkeypatch, tmp_path):
    """No usable kernel: KernelUnavailableError -> exit 2 (cli.py:151-154);
    never a silent CPU run."""
    from paper_2412_16370_b200 import kernels as K
    monkeypatch.setattr(K.B200Kernel, "available", lambda self: False)
    f = tmp_path / "x.bin"
    f.write_bytes(b"\x0f" * 8)
    code, _, err = run(capsys, "count", str(f))
    assert code == 2 and ("not available" in err or "no pospopcnt kernel" in err)
