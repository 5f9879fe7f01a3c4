#!/usr/bin/env python3
"""the paper's parameter studies on the same kernels.

* epsilon sweep at fixed minPts ("our methods tend to
  improve with increasing eps because there are fewer cells");
* minPts sweep 10 .. 10^4 at fixed eps (work for marking core
  points is O(n minPts));
* SS-varden, variable-density seed spreader, next to SS-simden.

Each line: JSON with the dataset, eps, minPts, device ms (CUDA events on the
launching stream, L2 flushed before each call, median of --reps), points/s,
per-stage ms and counters. Inputs are the BASELINE configs' generators.

usage: python tools/sweep.py [--n 10000000] [--reps 3] [--only eps|minpts|varden|qt|approx]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1912_06255_b200 as pkg  # noqa: E402


def timed(t, eps, mp, reps, flush, flags=0, rho=None):
    ms, last = [], None
    st = torch.cuda.current_stream()
    for _ in range(reps + 1):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        r = pkg.dbscan(t, eps, mp, flags=flags, timing=True, rho=rho)
        e1.record(st)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
        last = r
    return statistics.median(ms[1:]), last


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    flush = torch.empty(256 << 18, dtype=torch.int32, device="cuda")
    sets = []
    if a.only in ("", "eps"):
        ss3 = datagen.seed_spreader(a.n, 3, 1e6, 2, 1000 / a.n, noise_frac=1e-4)
        sets += [("ss-simden-3d", ss3, eps, 100) for eps in (250, 500, 1000, 2000, 4000)]
        uf = datagen.uniform(a.n, 3, 100_000, 4)
        sets += [("uniform-3d", uf, eps, 10) for eps in (250, 500, 1000, 2000)]
    if a.only in ("", "minpts"):
        ss3 = datagen.seed_spreader(a.n, 3, 1e6, 2, 1000 / a.n, noise_frac=1e-4)
        sets += [("ss-simden-3d", ss3, 1000, mp) for mp in (10, 100, 1000, 10_000)]
        uf = datagen.uniform(a.n, 3, 100_000, 4)
        sets += [("uniform-3d", uf, 500, mp) for mp in (10, 30, 100, 1000, 10_000)]
    if a.only in ("", "qt"):
        # row f2: minPts sweep where sparse points beside huge cells count long
        # (P:L1473-1477), plain scan vs per-cell trees (F_QUADTREE)
        ss3 = datagen.seed_spreader(a.n, 3, 1e6, 2, 1000 / a.n, noise_frac=1e-4)
        # default (sub-cell lower bounds from minPts 2000), without them, and
        # the per-point tree traversal (F_QUADTREE)
        for mp in (100, 1000, 3000, 10_000, 30_000):
            sets.append(("ss-simden-3d", ss3, 1000, mp))
            sets.append(("ss-simden-3d+noqb", ss3, 1000, mp))
            sets.append(("ss-simden-3d+qt", ss3, 1000, mp))
    if a.only in ("", "approx"):
        # row f4: rho-approximate DBSCAN on the same configs (rho = 0: exact)
        for cfgname in ("c3", "c4_7d"):
            cfg = datagen.CONFIGS[cfgname]
            pts = cfg.points()
            for rho in (0.0, 0.01, 0.1, 0.5, 1.0):
                sets.append((f"{cfgname}~rho={rho}", pts, cfg.eps, cfg.min_pts))
        # BCP-bound inputs: SS-simden 3D at eps = 4000 (large cells), uniform 3D
        # at eps = 1000 (sparse path) and 2000 (CSR path), all core
        ss3 = datagen.seed_spreader(a.n, 3, 1e6, 2, 1000 / a.n, noise_frac=1e-4)
        uf = datagen.uniform(a.n, 3, 100_000, 4)
        for rho in (0.0, 0.5, 1.0):
            sets.append((f"ss-simden-3d~rho={rho}", ss3, 4000, 100))
            sets.append((f"uniform-3d~rho={rho}", uf, 1000, 10))
            sets.append((f"uniform-3d~rho={rho}", uf, 2000, 10))
    if a.only in ("", "varden"):
        for d, L, eps in ((2, 1e6, 1000), (3, 1e6, 1000), (5, 1e5, 2000), (7, 1e5, 2000)):
            vd = datagen.seed_spreader(a.n, d, L, 20 + d, 1000 / a.n, varden=True)
            sets.append((f"ss-varden-{d}d", vd, eps, 100))
    for name, pts, eps, mp in sets:
        t = torch.from_numpy(pts).cuda()
        flags = pkg.F_QUADTREE if name.endswith("+qt") else (pkg.F_NO_QBOUND if name.endswith("+noqb") else 0)
        rho = float(name.split("rho=")[1]) if "~rho=" in name else 0.0
        ms, r = timed(t, eps, mp, a.reps, flush, flags, rho or None)
        print(json.dumps({"data": name, "n": len(pts), "d": pts.shape[1], "eps": eps, "min_pts": mp,
                          "ms": round(ms, 4), "pts_per_s": len(pts) / (ms / 1e3),
                          "stage_ms": {k: round(v, 4) for k, v in r.stage_ms.items()},
                          "stats": r.stats | {"n_core": r.n_core, "n_clusters": r.n_clusters,
                                              "n_border": r.n_border}}), flush=True)
        del t, r


if __name__ == "__main__":
    main()
