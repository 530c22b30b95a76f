#!/usr/bin/env python
"""Summarise one GPU session's ncu output (gpurun_out/<tag>/) into profiles/.

  python tools/ncu_summary.py <tag> <round-name>

Writes
  profiles/<round>_launches.csv       the launch list (kernel, grid, block, ns) of the
                                      bench command under `ncu --metrics gpu__time_duration.sum`
  profiles/<round>_ncu_summary.md     per-kernel-class share of the step (cold-cache,
                                      serialised launches) + the --set full key metrics
  profiles/ncu_traffic.json           DRAM bytes per k_spmv launch (read by bench.py's
                                      roofline "traffic" field)
"""
from __future__ import annotations

import csv
import io
import json
import os
import re
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes.sum.per_second", "DRAM bandwidth"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1 throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def read_csv_body(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    return list(csv.reader(io.StringIO("".join(lines))))


def kernel_class(name: str) -> str:
    m = re.search(r"topk::(k_\w+)", name) or re.search(r"\b(k_\w+)", name)
    return m.group(1) if m else "other (torch / library)"


def launches(tag_dir):
    rows = read_csv_body(os.path.join(tag_dir, "launches.csv"))
    hdr, data = rows[0], rows[1:]
    iname, ival = hdr.index("Kernel Name"), hdr.index("Metric Value")
    igrid, iblk = hdr.index("Grid Size"), hdr.index("Block Size")
    out = []
    for r in data:
        try:
            out.append((r[iname], r[igrid], r[iblk], float(r[ival])))
        except ValueError:
            pass
    return out


def full_metrics(tag_dir):
    res = {}
    for fn in sorted(os.listdir(tag_dir)):
        m = re.match(r"raw_(k_\w+)\.csv$", fn)
        if not m:
            continue
        rows = read_csv_body(os.path.join(tag_dir, fn))
        if len(rows) < 3:
            continue
        hdr, units, vals = rows[0], rows[1], rows[2]
        d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else m.group(1)}
        for key, label in KEYS:
            # exact column, else a section-prefixed one (e.g. "FBSP.TriageCompute.<key>")
            idx = hdr.index(key) if key in hdr else next((i for i, h in enumerate(hdr) if h.endswith("." + key)), None)
            if idx is not None:
                d[label] = (vals[idx], units[idx])
        res[m.group(1)] = d
    return res


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v) * mult


def main():
    tag, rnd = sys.argv[1], sys.argv[2]
    tag_dir = os.path.join(ROOT, "gpurun_out", tag)
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    md = [f"# ncu summary — {rnd} (gpurun_out/{tag})", ""]
    bench = os.path.join(tag_dir, "bench.log")
    if os.path.exists(bench):
        for ln in open(bench):
            if ln.startswith("{"):
                d = json.loads(ln)
                md += [f"bench: {d['value']:.1f} {d['unit']} ({d['ms_per_step']:.3f} ms/step), "
                       f"k_spmv {d['roofline']['achieved']:.0f} GB/s = {d['roofline']['frac']:.3f} of measured peak", ""]
    if os.path.exists(os.path.join(tag_dir, "launches.csv")):
        L = launches(tag_dir)
        with open(os.path.join(prof, f"{rnd}_launches.csv"), "w") as f:
            f.write("kernel,grid,block,ns\n")
            for n, g, b, ns in L:
                f.write(f"\"{n}\",\"{g}\",\"{b}\",{ns:.0f}\n")
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for n, _, _, ns in L:
            tot[kernel_class(n)] += ns
            cnt[kernel_class(n)] += 1
        ours = sum(v for k, v in tot.items() if k.startswith("k_"))
        md += ["## Launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)", "",
               "| kernel class | launches | total µs | share of our kernels |", "|---|---|---|---|"]
        for k in sorted(tot, key=lambda k: -tot[k]):
            share = f"{100 * tot[k] / ours:.1f}%" if k.startswith("k_") and ours else "—"
            md.append(f"| {k} | {cnt[k]} | {tot[k] / 1e3:.1f} | {share} |")
        md.append("")
    F = full_metrics(tag_dir)
    if F:
        md += ["## `ncu --set full` (one launch per kernel class)", ""]
        labels = [lab for _, lab in KEYS]
        md.append("| metric | " + " | ".join(F) + " |")
        md.append("|---|" + "---|" * len(F))
        for lab in labels:
            row = []
            for k in F:
                v = F[k].get(lab)
                row.append(f"{v[0]} {v[1]}".strip() if v else "—")
            md.append(f"| {lab} | " + " | ".join(row) + " |")
        md.append("")
        if "k_spmv" in F and "DRAM read" in F["k_spmv"]:
            r, w = F["k_spmv"]["DRAM read"], F["k_spmv"]["DRAM write"]
            traffic = to_bytes(*r) + to_bytes(*w)
            with open(os.path.join(prof, "ncu_traffic.json"), "w") as f:
                json.dump({"workload": "C3", "n_gpus": 1, "round": rnd, "source": f"gpurun_out/{tag}",
                           "spmv_dram_bytes_per_launch": traffic}, f, indent=1)
    with open(os.path.join(prof, f"{rnd}_ncu_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
