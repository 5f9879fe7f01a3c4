#!/usr/bin/env python3
"""Run one synthetic sweep instance through the C ABI (for ncu launch lists).
Usage: python tools/run_pts.py uniform|ss|varden N D eps minpts [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1912_06255_b200 as pkg  # noqa: E402

kind, n, d, eps, mp = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 2
if kind == "uniform":
    pts = datagen.uniform(n, d, 100_000, 4)
elif kind == "varden":  # tools/sweep.py's SS-varden instance
    pts = datagen.seed_spreader(n, d, 1e6 if d <= 3 else 1e5, 20 + d, 1000 / n, varden=True)
else:
    pts = datagen.seed_spreader(n, d, 1e6, 2, 1000 / n, noise_frac=1e-4)
t = torch.from_numpy(pts).cuda()
for i in range(reps):
    r = pkg.dbscan(t, eps, mp, timing=True)
    torch.cuda.synchronize()
print(kind, eps, mp, r.n_core, r.n_clusters, r.n_border, r.stats, {k: round(v, 3) for k, v in r.stage_ms.items()})
