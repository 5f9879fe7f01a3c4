#!/usr/bin/env python3
"""Top SASS instructions by warp-stall samples from an `ncu --page source
--csv --print-source sass` export (gzipped or not), per kernel.
usage: python tools/sass_hot.py file.csv[.gz] [kernel-substring] [top]"""
import csv
import gzip
import io
import sys

path = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
kern, hdr, rows, out = None, None, [], []
for r in csv.reader(raw):
    if r and r[0] == "Kernel Name":
        if kern and rows:
            out.append((kern, hdr, rows))
        kern, hdr, rows = r[1], None, []
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and r:
        rows.append(r)
if kern and rows:
    out.append((kern, hdr, rows))
for kern, hdr, rows in out:
    if want not in kern:
        continue
    ix = {h: i for i, h in enumerate(hdr)}
    S = ix["Warp Stall Sampling (All Samples)"]
    E = ix["Instructions Executed"]
    A = ix["Avg. Threads Executed"]
    tot_s = sum(int(r[S] or 0) for r in rows)
    tot_e = sum(int(r[E] or 0) for r in rows)
    print(f"== {kern[:100]}\n   stall samples {tot_s}, warp instructions {tot_e}")
    for n, r in sorted(enumerate(rows), key=lambda x: -int(x[1][S] or 0))[:top]:
        print(f"{n:5d} {int(r[S] or 0):7d} {int(r[E] or 0):10d} {r[A]:>6s}  {r[1].strip()[:70]}")


def ranges(path, want, cuts):
    """Executed warp instructions summed over SASS index ranges [cuts[i], cuts[i+1])."""
    raw = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    kern = hdr = None
    rows = []
    for r in csv.reader(raw):
        if r and r[0] == "Kernel Name":
            if kern and want in kern and rows:
                break
            kern, hdr, rows = r[1], None, []
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and r:
            rows.append(r)
    E = hdr.index("Instructions Executed")
    S = hdr.index("Warp Stall Sampling (All Samples)")
    for a, b in zip(cuts, cuts[1:]):
        print(f"[{a:5d},{b:5d}) exec {sum(int(r[E] or 0) for r in rows[a:b]):12d}  stalls {sum(int(r[S] or 0) for r in rows[a:b]):8d}")
