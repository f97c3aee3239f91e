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


def test_gpus_flag_without_gpus_fails_loudly():
    """--gpus 2 must launch two ranks on two sm_100 GPUs, never quietly
    measure one: with none visible it refuses (exit != 0, says why)."""
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--steps", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode != 0
    assert "visible sm_100" in res.stderr, res.stderr[-2000:]


def test_reference_arm_prints_the_gpu_arms_config():
    """Both arms describe the workload with the same dict (bench.config_dict),
    so the driver can match them; N comes from --gpus / WORLD_SIZE."""
    import importlib
    sys.path.insert(0, ROOT)
    bench = importlib.import_module("bench")
    code = (f"import sys; sys.path.insert(0, {ROOT!r}); sys.argv = ['bench.py', '--impl', "
            "'reference', '--gpus', '4', '--steps', '1', '--warmup', '3', '--config', 'c1']\n"
            "import bench; sys.exit(bench.main())\n")
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    mib2 = 2 << 20
    assert line["config"] == bench.config_dict("c1", 4, mib2, 4 * mib2, 16)
    assert line["n_gpus"] == 4 and line["cpu_baseline"]["host"]["cpu_model"]
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
