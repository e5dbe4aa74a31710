#!/usr/bin/env python
"""Summarise ncu output (run here, on the CPU box, over files gpurun brought back).

    python profiles/summarize_ncu.py --launches gpurun_out/launches.csv \
        --raw gpurun_out/prof.raw.csv --tag r01 [--steps 2 --warmup 1]

--launches: `ncu --metrics gpu__time_duration.sum --csv --log-file` output
--raw:      `ncu -i prof.ncu-rep --page raw --csv` output (one --set full capture)
Writes profiles/<tag>_launches.md, profiles/<tag>_kernels.md and updates
profiles/traffic.json (DRAM bytes per launch, read by bench.py's roofline).
"""
from __future__ import annotations

import argparse
import collections
import csv
import json
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))


def short(name: str) -> str:
    m = re.search(r"(k_[a-z0-9_]+)", name)
    base = m.group(1) if m else name[:40]
    t = re.search(r"k_[a-z0-9_]+<([^>]*)>", name)
    return f"{base}<{t.group(1)}>" if t else base


def launches(path: str, steps: int, out: str) -> None:
    text = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(text) if ln.startswith('"ID"'))  # skip ==PROF== lines
    rows = [r for r in csv.DictReader(text[start:]) if r.get("Metric Name") == "gpu__time_duration.sum"]
    per = collections.OrderedDict()
    for r in rows:
        k = short(r["Kernel Name"])
        v = float(r["Metric Value"])
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        per.setdefault(k, []).append(ns)
    total = sum(sum(v) for v in per.values())
    lines = ["| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / 1e3:.1f} | "
                     f"{100 * sum(v) / total:.1f}% |")
    with open(out, "w") as f:
        f.write(f"# ncu launch list ({os.path.basename(path)})\n\n")
        f.write("Cold-cache, serialised per-launch device times (`--metrics "
                "gpu__time_duration.sum --clock-control none`): compare shares, not absolutes.\n\n")
        f.write("\n".join(lines) + "\n")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def kernels(path: str, out: str) -> dict:
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    traffic = {}
    lines = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = short(d.get("Kernel Name", "?"))
        lines.append(f"## {name}\n")
        lines.append("| metric | value | unit |\n|---|---|---|")
        for k in WANT:
            if k in d:
                lines.append(f"| {k} | {d[k]} | {u.get(k, '')} |")
        try:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
            rb = float(d["dram__bytes_read.sum"]) * scale.get(u["dram__bytes_read.sum"], 1)
            wb = float(d["dram__bytes_write.sum"]) * scale.get(u["dram__bytes_write.sum"], 1)
            base = re.sub(r"<.*>", "", name)
            traffic.setdefault(base, int(rb + wb))
        except (KeyError, ValueError):
            pass
        lines.append("")
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary ({os.path.basename(path)})\n\n" + "\n".join(lines))
    return traffic


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--raw")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    if args.launches:
        launches(args.launches, args.steps, os.path.join(HERE, f"{args.tag}_launches.md"))
    if args.raw:
        t = kernels(args.raw, os.path.join(HERE, f"{args.tag}_kernels.md"))
        path = os.path.join(HERE, "traffic.json")
        old = json.load(open(path)) if os.path.exists(path) else {}
        old.update(t)
        json.dump(old, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
