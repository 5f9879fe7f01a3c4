#!/usr/bin/env python3
"""CPU baselines of SURVEY §8(d) / BASELINE.md §4, timed on the host cores of
the machine it runs on (the GPU box): O1 (brute force from the definition,
oracle/o1_bruteforce.c) single-threaded on c1 and on all cores on c2; O2 (the
simple CPU grid version, oracle/o2_grid.cpp) single-threaded and on all cores
on every BASELINE run. The oracles are run as they stand (test
infrastructure, never tuned). One JSON line per measurement, each in its own
subprocess so that OMP_NUM_THREADS takes effect.

usage: python tools/cpu_baselines.py [--runs c1,c2,...] [--skip-o1]"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(kind, name, threads):
    import numpy as np  # noqa: F401
    import datagen
    import oracle
    oracle.build()
    cfg = datagen.CONFIGS[name]
    pts = cfg.points()
    sha = datagen.sha256_prefix(pts)
    t0 = time.perf_counter()
    if kind == "o1":
        r = oracle.o1(pts, cfg.eps, cfg.min_pts, threads=threads)
    else:
        r = oracle.o2(pts, cfg.eps, cfg.min_pts)
    dt = time.perf_counter() - t0
    print(json.dumps({"oracle": kind.upper(), "run": name, "n": cfg.n, "d": cfg.d, "eps": cfg.eps,
                      "min_pts": cfg.min_pts, "threads": threads, "seconds": round(dt, 3),
                      "points_per_s": cfg.n / dt, "n_core": int(r.core.sum()), "nnz": int(len(r.border_ids)),
                      "sha256_16": sha}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", default="c1,c2,c3,c4_5d,c4_7d,c5_10,c5_10k")
    ap.add_argument("--skip-o1", action="store_true")
    ap.add_argument("--one", nargs=3, metavar=("KIND", "RUN", "THREADS"))
    args = ap.parse_args()
    if args.one:
        return one(args.one[0], args.one[1], int(args.one[2]))
    nproc = os.cpu_count()
    model = ""
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    print(json.dumps({"host": {"nproc": nproc, "lscpu_model": model}}), flush=True)
    jobs = []
    if not args.skip_o1:
        jobs += [("o1", "c1", 1), ("o1", "c2", nproc)]
    for r in args.runs.split(","):
        jobs += [("o2", r, 1), ("o2", r, nproc)]
    for kind, name, th in jobs:
        env = dict(os.environ, OMP_NUM_THREADS=str(th))
        subprocess.run([sys.executable, __file__, "--one", kind, name, str(th)], env=env, check=False)


if __name__ == "__main__":
    main()
