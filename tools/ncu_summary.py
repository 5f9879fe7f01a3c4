#!/usr/bin/env python3
"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch) into
per-kernel totals and shares. Usage: python tools/ncu_summary.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
for r in rows:
    if not r:
        continue
    if r[0] == "ID":
        hdr = r
        continue
    if hdr is None:
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} share")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:40s} {v[0]:8d} {v[1]:12.1f} {v[1] / v[0]:10.2f} {v[1] / tot:6.1%}")
print(f"{'TOTAL':40s} {sum(v[0] for v in agg.values()):8d} {tot:12.1f}")
