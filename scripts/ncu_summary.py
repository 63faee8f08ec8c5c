#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python scripts/ncu_summary.py --full gpurun_out/prof_<wl>_<prec>.ncu-rep ... \
        --launches gpurun_out/launches.csv --tag r01

Writes profiles/ncu_summary.json (per workload/precision: duration, DRAM bytes,
tensor-pipe and issue utilisation, registers, ...) — bench.py reads the DRAM
traffic from it — and profiles/ncu_<tag>.md (human readable, with the launch
list's per-kernel share of the step)."""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import re
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "duration_ms": "gpu__time_duration.sum",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "lts_bytes": "lts__t_bytes.sum",
    "tensor_pipe_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    # tensor memory (TMEM) activity: the epilogue / final-layer reads co-limit the 16-bit kernel
    "tmem_active_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "registers_per_thread": "launch__registers_per_thread",
    "grid_size": "launch__grid_size",
    "block_size": "launch__block_size",
    "smem_dynamic_bytes": "launch__shared_mem_per_block_dynamic",
    "warp_instructions": "smsp__inst_executed.sum",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6, "s": 1e3,
         "Ghz": 1, "Mhz": 1e-3}


def raw(rep):
    """Rows of `ncu -i <rep> --page raw --csv`; a `.raw.csv` file exported on
    the GPU box (the .ncu-rep files exceed gpurun's copy-back limit) is read as is."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for key, metric in METRICS.items():
            if metric in hdr:
                i = hdr.index(metric)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                d[key] = v * SCALE.get(units[i], 1)
        d["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        res.append(d)
    return res


def launches(path):
    """Per-kernel total time share from a --metrics gpu__time_duration.sum --csv log."""
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = defaultdict(lambda: [0.0, 0])
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki]).strip()
        v = float(r[vi].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(r[ui], 1.0)
        per[name][0] += v
        per[name][1] += 1
    return per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--launches", default=None)
    ap.add_argument("--tag", default="r01")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    js_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(js_path)) if os.path.exists(js_path) else {}
    md = [f"# ncu summary ({a.tag})", ""]
    for rep in a.full:
        m = re.search(r"prof\w*?_([a-z0-9]+)_([a-z0-9]+)\.(?:ncu-rep|raw\.csv)$", os.path.basename(rep))
        key = f"{m.group(1)}/{m.group(2)}" if m else os.path.basename(rep)
        for d in raw(rep):
            if "sweep_kernel" not in d["kernel"]:
                continue
            d["dram_bytes_per_launch"] = d.get("dram_read_bytes", 0) + d.get("dram_write_bytes", 0)
            d["source"] = os.path.basename(rep)
            d["tag"] = a.tag
            summary[key] = d
            md.append(f"## {key} — `{d['kernel'][:80]}` (ncu --set full, --clock-control none, one launch)")
            for k2 in ["duration_ms", "sm_clock_ghz", "tensor_pipe_active_pct", "tmem_active_pct", "issue_active_pct", "alu_pipe_pct",
                       "fma_pipe_pct", "dram_bytes_per_launch", "lts_bytes", "registers_per_thread", "grid_size",
                       "block_size", "smem_dynamic_bytes", "warp_instructions"]:
                if k2 in d:
                    md.append(f"- {k2}: {d[k2]:.6g}" if isinstance(d[k2], float) else f"- {k2}: {d[k2]}")
            md.append("")
    if a.launches and os.path.exists(a.launches):
        per = launches(a.launches)
        tot = sum(v[0] for v in per.values())
        md.append("## Launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)")
        md.append("")
        md.append("| kernel | launches | total ms | share |")
        md.append("|---|---|---|---|")
        for name, (ms, n) in sorted(per.items(), key=lambda x: -x[1][0]):
            md.append(f"| {name} | {n} | {ms:.3f} | {ms / tot:.1%} |")
        summary[f"launches_{a.tag}"] = {n: {"ms": v[0], "launches": v[1], "share": v[0] / tot} for n, v in per.items()}
    json.dump(summary, open(js_path, "w"), indent=1)
    with open(os.path.join(ROOT, "profiles", f"ncu_{a.tag}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
