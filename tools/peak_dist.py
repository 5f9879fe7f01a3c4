#!/usr/bin/env python3
"""U1 `peak_dist` sweep: measured exact distance tests
per second on this GPU for d = 2, 3, 5, 7, the three predicate variants
(0 shipped uint32, 1 shipped 64-bit, 2 fp64) and register tiles of 1, 2, 4
queries per thread. One JSON line per point; the maximum over tiles of the
uint32 variant at the run's d is the a6/a8 roofline denominator (bench.py
measures d = 3 live as well)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1912_06255_b200 as pkg  # noqa: E402


def main():
    torch.cuda.init()
    for d in (2, 3, 5, 7):
        for v in (0, 1, 2):
            for qt in (1, 2, 4):
                reps = 200 if v != 2 else 20
                r = pkg.peak_dist(d, v, qt, reps)
                r["T_tests_per_s"] = round(r["tests_per_s"] / 1e12, 4)
                r["hit_frac"] = round(r["hits"] / r["tests"], 4)
                print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
