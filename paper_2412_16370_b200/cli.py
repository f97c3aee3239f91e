"""Command line: ``count``, ``selftest`` and ``kernels`` of the reference CLI
over the B200 kernel (/root/reference/pkg/src/pospopcnt/cli.py:46-58, 82-94,
134-158; selftest.py:44-90).

    python -m paper_2412_16370_b200 count [--width W] [--format lines|csv] [FILE]
    python -m paper_2412_16370_b200 selftest [--seed S] [--iterations N]
    python -m paper_2412_16370_b200 kernels

Same arguments, output and exit status as the reference (0 success, 2 usage
or input errors, incl. no usable GPU).  A FILE is memory-mapped rather than
read into a bytes object (cli.py:84-85 reads it whole): the pages go straight
into pp_count_host's pinned staging ring, overlapped with the H2D copies and
the counting.  The reference's ``bench`` / ``selftest`` subcommands are
measurement layer (bench.py at the repo root is this build's benchmark);
``selftest`` is restated: random widths, lengths and offsets, the kernel
against the reference's scalar definition (``scalar_pospopcnt``, the public
API's checker -- never a fallback), on host bytes and on CUDA tensors, with
the reference's shrink-to-minimal-case report on a mismatch.
"""

import argparse
import os
import random
import sys

import numpy as np

from .core import (
    WORD_WIDTHS,
    InputLengthError,
    InputView,
    KernelUnavailableError,
    UnknownKernelError,
    new_counters,
    scalar_pospopcnt,
)
from .kernels import list_kernels, pospopcnt, select_kernel


def build_parser():
    parser = argparse.ArgumentParser(
        prog="pospopcnt-b200",
        description="Positional population counts on a B200: per-bit-position "
        "set-bit counters over arrays of 8/16/32/64-bit words.")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("count", help="count a file (or stdin)")
    p.add_argument("--width", type=int, choices=WORD_WIDTHS, default=8)
    p.add_argument("--kernel", default=None, help="kernel name (default: auto)")
    p.add_argument("--format", choices=("lines", "csv"), default="lines")
    p.add_argument("file", nargs="?", help="input file (default: stdin)")
    p = sub.add_parser("selftest", help="randomized correctness check")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--iterations", type=int, default=1000)
    sub.add_parser("kernels", help="list kernels and availability")
    return parser


_BIG = 65536  # every 16th case: up to 64 KiB (selftest.py:56-58)
_SMALL = 4096


def _case_run(kernel, data, offset, length, w, device):
    if device:
        import torch
        data = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda() if data else \
            torch.zeros(0, dtype=torch.uint8, device="cuda")
    return kernel.run(InputView(data, offset, length), w, new_counters(w))


def _shrink(kernel, data, offset, length, w, device):
    """Greedily halve the failing input while the mismatch persists
    (selftest.py:20-41)."""
    step = w // 8

    def bad(off, ln):
        return _case_run(kernel, data, off, ln, w, device) != scalar_pospopcnt(
            InputView(data, off, ln), w)

    changed = True
    while changed and length > step:
        changed = False
        half = (length // 2) // step * step
        if half and bad(offset, half):
            length = half
            changed = True
            continue
        if half and bad(offset + (length - half), half):
            offset += length - half
            length = half
            changed = True
    return offset, length


def run_selftest(iterations=1000, seed=1, out=print):
    """The reference's randomized self-test (selftest.py:44-90) for the B200
    kernel; even cases count host bytes (pp_count_host), odd ones a CUDA
    tensor (pp_count_sync).  Returns True when every case agreed."""
    rng = random.Random(seed)
    kernel = select_kernel()
    host_cases = device_cases = 0
    for case in range(iterations):
        w = rng.choice(WORD_WIDTHS)
        step = w // 8
        limit = _BIG if case % 16 == 15 else _SMALL
        length = rng.randrange(0, limit // step + 1) * step
        offset = rng.randrange(64)
        data = rng.randbytes(offset + length + rng.randrange(8))
        device = case % 2 == 1
        got = _case_run(kernel, data, offset, length, w, device)
        want = scalar_pospopcnt(InputView(data, offset, length), w)
        device_cases += device
        host_cases += not device
        if got != want:
            m_off, m_len = _shrink(kernel, data, offset, length, w, device)
            where = "cuda tensor" if device else "host bytes"
            out(f"selftest: MISMATCH kernel={kernel.name} ({where}) vs scalar oracle "
                f"width={w} length={m_len} offset={m_off} seed={seed} case={case}")
            out(f"selftest: reproduce with length={m_len} offset={m_off} "
                f"width={w} seed={seed}")
            return False
    out(f"selftest: PASS ({host_cases} host-buffer cases, {device_cases} device cases, "
        f"seed={seed})")
    return True


def cmd_selftest(args):
    return 0 if run_selftest(iterations=args.iterations, seed=args.seed) else 1


def _file_bytes(path):
    """The file's bytes without a copy: a read-only memory map (empty files
    cannot be mapped: an empty buffer)."""
    if os.path.getsize(path) == 0:
        with open(path, "rb"):  # still raise for unreadable paths
            return b""
    return np.memmap(path, dtype=np.uint8, mode="r")


def cmd_count(args):
    data = _file_bytes(args.file) if args.file else sys.stdin.buffer.read()
    counters = pospopcnt(data, args.width, kernel=args.kernel)
    if args.format == "csv":
        print(",".join(str(v) for v in counters))
    else:
        for v in counters:
            print(v)
    return 0


def cmd_kernels(_args):
    for desc, ok in list_kernels():
        flag = "available" if ok else "unavailable"
        print(f"{desc.name:10s} r={desc.r:<6d} block={desc.block_bytes:<7d} {flag}")
    return 0


def main(argv=None):
    args = build_parser().parse_args(argv)
    handler = {"count": cmd_count, "selftest": cmd_selftest,
               "kernels": cmd_kernels}[args.command]
    try:
        return handler(args)
    except (InputLengthError, UnknownKernelError, KernelUnavailableError,
            ValueError, OSError) as exc:
        print(f"pospopcnt-b200: error: {exc}", file=sys.stderr)
        return 2
    except KeyboardInterrupt:
        return 1


if __name__ == "__main__":
    sys.exit(main())
