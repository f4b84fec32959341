#!/usr/bin/env python
"""Summarises ncu captures into profiles/ (tracked).

    python scripts/ncu_summary.py --launches gpurun_out/r01_launches.csv \
        --full gpurun_out/r01_full.ncu-rep --tag r01 --config 2

Writes profiles/<tag>_launches.md (per-kernel device time, cold-cache,
serialised: compare SHARES), profiles/<tag>_ncu_full.md (key metrics of the
--set full capture) and updates profiles/union_kernel_ncu.json with the
union kernel's DRAM bytes per launch (bench.py reports it as `traffic`).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROFILES = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data-pipe wavefronts % peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput % peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % peak"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % peak"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_throttle / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not_selected / issue"),
]


def launches(path, tag, command):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    lines = [f"# {tag}: kernel launch list (ncu --metrics gpu__time_duration.sum --clock-control none)",
             "", "Cold-cache, serialised replay of `" + command + "` "
             "(engine builds, seeding and flushes included): compare shares, "
             "not absolutes.", "", "| kernel | launches | mean µs | min µs |", "|---|---|---|---|"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v)/len(v)/1e3:.1f} | {min(v)/1e3:.1f} |")
    return "\n".join(lines) + "\n"


def full(path, tag):
    if path.endswith(".csv"):  # `ncu -i rep --page raw --csv` exported on the GPU box
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out, per_kernel = [], {}
    for row in rows[2:]:
        name = row[hdr.index("Kernel Name")]
        m = {}
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                m[label] = (row[i], units[i])
        per_kernel.setdefault(name.split("(")[0], []).append(m)
    out.append(f"# {tag}: ncu --set full (--clock-control none), per launch\n")
    for k, ms in per_kernel.items():
        out.append(f"## `{k}`\n")
        out.append("| metric | " + " | ".join(f"launch {i}" for i in range(len(ms))) + " |")
        out.append("|---|" + "---|" * len(ms))
        for _, label in KEYS:
            vals = [m.get(label, ("", ""))for m in ms]
            out.append(f"| {label} | " + " | ".join(f"{v} {u}".strip() for v, u in vals) + " |")
        out.append("")
    return "\n".join(out) + "\n", per_kernel


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--command", default="python bench.py --steps 2 --warmup 1")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--sum-launches", action="store_true",
                    help="the captured launches are one step (item sweep + main sweep of a "
                         "source-blocked dense step): record their summed DRAM bytes")
    a = ap.parse_args()
    os.makedirs(PROFILES, exist_ok=True)
    if a.launches:
        with open(os.path.join(PROFILES, f"{a.tag}_launches.md"), "w") as f:
            f.write(launches(a.launches, a.tag, a.command))
    if a.full:
        text, per = full(a.full, a.tag)
        with open(os.path.join(PROFILES, f"{a.tag}_ncu_full.md"), "w") as f:
            f.write(text)
        union = [k for k in per if "union_kernel" in k]
        if union:
            ms = per[union[0]]

            def num(m, label):
                v, u = m[label]
                v = float(v.replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

            traffic = sum(num(m, "DRAM read") + num(m, "DRAM write") for m in ms)
            if not a.sum_launches:
                traffic /= len(ms)
            path = os.path.join(PROFILES, "union_kernel_ncu.json")
            doc = json.load(open(path)) if os.path.exists(path) else {}
            doc[f"config{a.config}"] = {"dram_bytes_per_launch": traffic, "source": f"{a.tag}_ncu_full.md",
                                        "kernel": union[0]}
            if a.sum_launches:
                doc[f"config{a.config}"]["note"] = (f"sum of the {len(ms)} launches of one "
                                                    "source-blocked dense step")
            json.dump(doc, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
