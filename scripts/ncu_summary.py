#!/usr/bin/env python3
"""Summarise an ncu --set full report + a launch-list CSV into profiles/.

  python scripts/ncu_summary.py REPORT.ncu-rep LAUNCHES.csv OUT_PREFIX
writes OUT_PREFIX_ncu_summary.md, OUT_PREFIX_launches.csv and updates
profiles/ncu_traffic.json (dram bytes per launch of each hot kernel).
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__bytes_read.sum.per_second", "dram read BW"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1tex %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("smsp__inst_executed.sum", "warp instructions"),
]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def short(name):
    for w in (8, 16, 32, 64):  # categories kernels carry a third (code-bytes) parameter
        if f"pp_tma_kernel<{w}, 16, 1>" in name:
            return f"pp_tma_kernel<{w}, 16>"
    for k in ("pp_tma_kernel<32, 16>", "pp_tma_kernel<8, 16>", "pp_tma_kernel<16, 16>",
              "pp_tma_kernel<64, 16>", "pp_tma_kernel<1,", "pp_tma_kernel<0,",
              "pp_tma_kernel<1>", "pp_tma_kernel<0>", "pp_tma_kernel<true>", "pp_tma_kernel<false>",
              "pp_segtma_kernel<8>", "pp_seg_kernel<8>", "pp_seg_kernel", "pp_cat_kernel<1>", "pp_count_ldg_kernel", "gen_"):
        if k in name:
            return {"pp_tma_kernel<true>": "pp_tma_kernel<1>", "pp_tma_kernel<1,": "pp_tma_kernel<1>",
                    "pp_tma_kernel<false>": "pp_tma_kernel<0>", "pp_tma_kernel<0,": "pp_tma_kernel<0>",
                    "pp_seg_kernel<8>": "pp_seg_kernel"}.get(k, k)
    return name[:40]


def main(rep, launches, prefix):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = [f"# ncu --set full summary: {os.path.basename(rep)}", "",
           "Captured with `ncu --set full --clock-control none --import-source on -k regex:pp_` "
           "on one B200 (sm_100a), 1 GiB inputs (scripts/prof_kernels.py).", ""]
    traffic = {}
    for r in rows[2:]:
        name = short(r[hdr.index("Kernel Name")])
        out.append(f"## {name}")
        out.append("")
        out.append("| metric | value |")
        out.append("|---|---|")
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"| {label} (`{k}`) | {r[i]} {units[i]} |")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith(STALLS) and not h.endswith("not_issued"):
                try:
                    st.append((float(r[i]), h[len(STALLS):]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        out.append("")
        out.append("top stall reasons (pc sampling): " + ", ".join(
            f"{n} {100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:5]))
        out.append("")
        rd = r[hdr.index("dram__bytes_read.sum")]
        wr = r[hdr.index("dram__bytes_write.sum")]
        ur = units[hdr.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(ur, 1)
        uw = units[hdr.index("dram__bytes_write.sum")]
        scw = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(uw, 1)
        traffic.setdefault(name, {"bytes": int(float(rd) * scale + float(wr) * scw),
                                  "input_bytes": 1 << 30})
    with open(prefix + "_ncu_summary.md", "w") as f:
        f.write("\n".join(out) + "\n")
    # launch list: keep the per-launch rows
    if launches and os.path.exists(launches):
        lines = open(launches).read().splitlines()
        start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
        with open(prefix + "_launches.csv", "w") as f:
            f.write("\n".join(lines[start:]) + "\n")
    tj = os.path.join(os.path.dirname(prefix), "ncu_traffic.json")
    d = json.load(open(tj)) if os.path.exists(tj) else {}
    d.update(traffic)
    d["_source"] = os.path.basename(prefix) + "_ncu_summary.md (dram__bytes_read.sum + "\
        "dram__bytes_write.sum per launch, 1 GiB input)"
    json.dump(d, open(tj, "w"), indent=1)
    print(open(prefix + "_ncu_summary.md").read())


if __name__ == "__main__":
    main(*sys.argv[1:4])
