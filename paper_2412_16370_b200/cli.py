"""Command line: ``count`` and ``kernels`` of the reference CLI over the B200
kernel (/root/reference/pkg/src/pospopcnt/cli.py:46-58, 82-94, 134-158).

    python -m paper_2412_16370_b200 count [--width W] [--format lines|csv] [FILE]
    python -m paper_2412_16370_b200 kernels

Same arguments, output and exit status as the reference (0 success, 2 usage
or input errors, incl. no usable GPU).  A FILE is memory-mapped rather than
read into a bytes object (cli.py:84-85 reads it whole): the pages go straight
into pp_count_host's pinned staging ring, overlapped with the H2D copies and
the counting.  The reference's ``bench`` / ``selftest`` subcommands are
its measurement and test layer, not restated here: with the b200 kernel
registered into the reference (ref_plugin.register), the reference's own
selftest and bench drive it (tests/test_gpu_ref_hw.py); bench.py at the repo
root is this build's benchmark.
"""

import argparse
import os
import sys

import numpy as np

from .core import WORD_WIDTHS, InputLengthError, KernelUnavailableError, UnknownKernelError
from .kernels import list_kernels, pospopcnt


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
    sub.add_parser("kernels", help="list kernels and availability")
    return parser


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
    handler = {"count": cmd_count, "kernels": cmd_kernels}[args.command]
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
