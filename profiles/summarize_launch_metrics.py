#!/usr/bin/env python
"""Summarise an ncu launch list captured with
`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`
(cold-cache, serialised launches): per kernel, launches, mean device time,
mean DRAM bytes per launch and the share of the listed time.

    python profiles/summarize_launch_metrics.py gpurun_out/r2h_launches_n1.csv \
        --title "..." --out profiles/r02_launches_n1.md [--only regex]
"""
from __future__ import annotations

import argparse
import collections
import csv
import re

SCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
         "s": 1.0, "second": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(name: str) -> str:
    m = re.search(r"(k_[a-z0-9_]+)", name)
    base = m.group(1) if m else name[:48]
    t = re.search(r"k_[a-z0-9_]+<([^>]*)>", name)
    return f"{base}<{t.group(1)}>" if t else base


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--title", default="")
    ap.add_argument("--out", required=True)
    ap.add_argument("--only", default=None, help="regex on the short kernel name")
    a = ap.parse_args()
    text = open(a.csv).read().splitlines()
    start = next(i for i, ln in enumerate(text) if ln.startswith('"ID"'))
    launches = collections.OrderedDict()
    for r in csv.DictReader(text[start:]):
        key = (r["ID"], r["Kernel Name"])
        d = launches.setdefault(key, {})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * SCALE.get(r.get("Metric Unit", ""), 1.0)
    per = collections.OrderedDict()
    for (_, name), d in launches.items():
        k = short(name)
        if a.only and not re.search(a.only, k):
            continue
        e = per.setdefault(k, [0, 0.0, 0.0, 0.0])
        e[0] += 1
        e[1] += d.get("gpu__time_duration.sum", 0.0)
        e[2] += d.get("dram__bytes_read.sum", 0.0)
        e[3] += d.get("dram__bytes_write.sum", 0.0)
    total = sum(e[1] for e in per.values()) or 1.0
    lines = [f"# {a.title}", "",
             f"From `{a.csv.split('/')[-1]}`: ncu `--metrics gpu__time_duration.sum,dram__bytes_read.sum,"
             "dram__bytes_write.sum --clock-control none` (cold-cache, serialised launches: compare "
             "shares and bytes, not absolute times).", "",
             "| kernel | launches | mean us | DRAM read GB/launch | DRAM write GB/launch | GB/s | share |",
             "|---|---|---|---|---|---|---|"]
    for k, (n, t, rd, wr) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        mt = t / n
        gbs = (rd + wr) / n / mt / 1e9 if mt > 0 else 0.0
        lines.append(f"| {k} | {n} | {mt * 1e6:.1f} | {rd / n / 1e9:.4f} | {wr / n / 1e9:.4f} | {gbs:.0f} | "
                     f"{t / total * 100:.1f}% |")
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
