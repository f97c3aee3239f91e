"""bench.py's output contract on the CPU side: the reference arm prints
exactly one JSON line on stdout, whatever else writes to fd 1."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_one_json_line():
    # a stray write to fd 1 from "a library" (here: a sitecustomize-free
    # trick -- python -c that imports bench and prints before and after)
    code = (
        "import os, sys, runpy\n"
        f"sys.path.insert(0, {ROOT!r})\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', '--steps', '1',"
        " '--warmup', '3']\n"
        "import bench\n"
        "bench.claim_stdout()\n"
        "os.write(1, b'NCCL version 0.0.0 (chatter on fd 1)\\n')\n"
        "sys.exit(bench.main())\n")
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    out = [x for x in res.stdout.splitlines() if x.strip()]
    assert len(out) == 1, res.stdout
    line = json.loads(out[0])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    assert "NCCL version" in res.stderr
