"""bench.py's JSON line carries every key of the driver's contract (and the
reference arm's), with consistent values -- run on the GPU box."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    out = [x for x in res.stdout.splitlines() if x.strip()]
    assert len(out) == 1, res.stdout
    return json.loads(out[0])


def test_bench_line_contract(cuda):
    d = _run("--steps", "5", "--warmup", "3", "--cpu-min-time", "0.5")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True and d["dtype"] == "u8"
    assert d["value"] > 1000 and d["exact"] is True
    # C2 is per-GPU work (weak scaling), whatever objects ride along (strong_c5)
    assert d["scaling"] == "weak"
    assert abs(d["value"] - d["config"]["bytes_per_step_all_gpus"] / d["ms_per_step"] / 1e6) \
        < 0.01 * d["value"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    c = d["cpu_baseline"]
    assert c["kind"] in ("reference", "port") and c["cores"] >= 1 and c["value"] > 0
    assert c["sample"] and c["host"]["cpu_model"]
    if c["kind"] == "reference":  # baseline/_ref shipped: BASELINE.md section 3 rows
        assert {"ref-numba-1core", "ref-numba-Pcore", "ref-default", "ref-scalar"} <= \
            set(c["rows"])
        assert c["one_core"] > 0 and c["rows"]["ref-default"]["kernel"] == "numpy"
    s = d["strong_c5"]
    assert s["exact"] is True and s["bytes_total"] == 64 << 30 and s["value"] > 1000
    e = d["e2e"]
    assert e["unit"] == "GB/s" and e["value"] > 0
    assert e["h2d_bytes_per_step"] == d["config"]["bytes_per_gpu_per_step"]
    assert e["d2h_bytes_per_step"] > 0
    # the same public call on pageable memory (bytes / numpy callers)
    assert d["e2e_pageable"]["unit"] == "GB/s" and d["e2e_pageable"]["value"] > 0
    assert d["gpu_launches"] == 5
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert "workload" in d["config"]
    # every other BASELINE config measured in the same run, each exact
    oc = d["other_configs"]
    assert set(oc) == {"c1", "c3", "c4", "c4seg", "c3cat"}, oc
    for name, o in oc.items():
        assert "error" not in o, (name, o)
        assert o["exact"] is True and o["value"] > 0, (name, o)
    assert oc["c3cat"]["roofline"]["bound"] == "alu"
    assert oc["c1"]["cold_call"]["us_median"] > 0


def test_reference_arm_contract():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "3")
    g = _run("--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu-baseline",
             "--no-strong-c5", "--no-all-configs")
    # same workload description as the GPU arm: the driver matches the lines
    assert d["config"] == g["config"] and d["metric"] == g["metric"]
    assert d["scaling"] == g["scaling"] == "weak"
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["cpu_baseline"]["value"] == d["value"] and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["gpu_launches"] == 0
