"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`)
into a markdown table of kernels by total time.
Usage: python tools/launch_summary.py launches.csv out.md [title]"""
import csv
import sys
from collections import defaultdict

src, dst = sys.argv[1], sys.argv[2]
title = sys.argv[3] if len(sys.argv) > 3 else src
lines = open(src, encoding="utf-8", errors="replace").read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
agg = defaultdict(lambda: [0, 0.0])
for row in csv.DictReader(lines[start:]):
    if row["Metric Name"] != "gpu__time_duration.sum":
        continue
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(row["Metric Unit"], 1e-3)
    a = agg[row["Kernel Name"][:70]]
    a[0] += 1
    a[1] += float(row["Metric Value"].replace(",", "")) * scale
total = sum(v[1] for v in agg.values())
out = [f"# {title}", "", "Cold-cache, serialised per-launch times; compare shares, not absolutes.", "",
       "| kernel | launches | mean us | total us |", "|---|---|---|---|"]
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"| {k} | {n} | {t / n:.1f} | {t:.1f} ({100 * t / total:.1f}%) |")
open(dst, "w").write("\n".join(out) + "\n")
print("\n".join(out))
