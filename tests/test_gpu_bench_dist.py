"""bench.py's N>1 path, two ranks on one GPU (gloo, test hooks).

The driver runs `bench.py` under torchrun at N = 2, 4, 8 on a multi-GPU box;
this run has one GPU.  PP_BENCH_DEVICE=0 puts both ranks on cuda:0 and
PP_BENCH_BACKEND=gloo replaces NCCL (which refuses two ranks on one
device).  The ranks' kernels never wait on one another -- with the fused
exchange each only issues atomics into the other's IPC-mapped counters -- so
the code path is the real one: handle exchange, pp_count_multi steps, the
max-over-ranks timing, and the exactness check of the job total (every
rank's oracle count summed, C2; the reference's own 64 GiB total, C5).
Timings from such a run mean nothing and are not reported anywhere.
"""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("config,exchange", [("c2", "fused"), ("c2", "nccl"), ("c5", "fused")])
def test_bench_two_ranks_one_gpu(cuda, config, exchange):
    env = dict(os.environ, PP_BENCH_DEVICE="0", PP_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--config", config, "--exchange", exchange, "--no-e2e", "--no-cpu-baseline"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    # stdout carries exactly one line, the JSON (NCCL / torch chatter -> stderr)
    out = [x for x in res.stdout.splitlines() if x.strip()]
    assert len(out) == 1 and out[0].startswith("{"), res.stdout[-3000:]
    lines = [json.loads(out[0])]
    line = lines[0]
    assert line["n_gpus"] == 2 and line["exact"] is True, line
    assert line["config"]["bytes_per_step_all_gpus"] == (
        2 * line["config"]["bytes_per_gpu_per_step"] if config == "c2" else 64 << 30)
    if config == "c2":  # the 64 GiB C5 array split over the two ranks, exact
        sc = line["strong_c5"]
        assert sc["exact"] is True and sc["n_gpus"] == 2 and sc["bytes_per_gpu"] == 32 << 30


def test_bench_gpus_flag_relaunches_ranks(cuda):
    """`bench.py --gpus 2` outside torchrun launches the two ranks itself
    (same command shape as the driver's) and reports n_gpus = 2."""
    env = dict(os.environ, PP_BENCH_DEVICE="0", PP_BENCH_BACKEND="gloo")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--no-cpu-baseline"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    out = [x for x in res.stdout.splitlines() if x.strip()]
    assert len(out) == 1 and out[0].startswith("{"), res.stdout[-3000:]
    line = json.loads(out[0])
    assert line["n_gpus"] == 2 and line["exact"] is True and line["strong_c5"]["exact"] is True
    assert line["config"]["bytes_per_step_all_gpus"] == 2 << 30
    # e2e at N ranks: every rank's host shard through pospopcnt_sharded
    e = line["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 1 << 30 and "sharded" in e["path"]


def test_bench_gpus_mismatch_fails_loudly(cuda):
    """Under torchrun, --gpus must equal the world size; and --gpus N with
    fewer than N GPUs visible refuses to run instead of measuring one GPU."""
    import torch
    n = torch.cuda.device_count()
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n + 1),
                          "--steps", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode != 0 and "visible sm_100" in res.stderr
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--steps", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env=env)
    assert res.returncode != 0 and "WORLD_SIZE=1" in res.stderr
