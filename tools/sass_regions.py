#!/usr/bin/env python3
"""Stall samples / executed warp instructions of one kernel's SASS, split at
barriers (BAR.SYNC) and listed by the hottest instructions per region.
usage: python tools/sass_regions.py file.csv[.gz] [top]"""
import csv
import gzip
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 6
rows, hdr = [], None
for r in csv.reader(gzip.open(path, "rt") if path.endswith(".gz") else open(path)):
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and r and r[0] != "Kernel Name":
        rows.append(r)
S = hdr.index("Warp Stall Sampling (All Samples)")
E = hdr.index("Instructions Executed")
A = hdr.index("Avg. Threads Executed")
stall = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
cuts = [0] + [i + 1 for i, r in enumerate(rows) if "BAR.SYNC" in r[1] or "TRYWAIT" in r[1]] + [len(rows)]
ts = sum(int(r[S] or 0) for r in rows)
te = sum(int(r[E] or 0) for r in rows)
print(f"total stall samples {ts}, warp instructions {te}")
for a, b in zip(cuts, cuts[1:]):
    s = sum(int(r[S] or 0) for r in rows[a:b])
    if s < 0.02 * ts:
        continue
    e = sum(int(r[E] or 0) for r in rows[a:b])
    why = sorted(((sum(int(r[hdr.index(h)] or 0) for r in rows[a:b]), h) for h in stall), reverse=True)[:3]
    print(f"[{a}:{b}) samples {s} ({100*s/ts:.0f}%) instr {e} ({100*e/te:.0f}%)  " + ", ".join(f"{h[6:]} {v}" for v, h in why))
    for i in sorted(range(a, b), key=lambda i: -int(rows[i][S] or 0))[:top]:
        r = rows[i]
        print(f"   {i:5d} {r[S]:>6s} {r[E]:>10s} {r[A]:>3s}  {r[1].strip()[:64]}")
