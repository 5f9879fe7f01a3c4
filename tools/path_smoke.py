#!/usr/bin/env python3
"""Small calls over every path (CSR, all-pairs, tree, sparse brick / brick
overflow / thread, 1D-2D, radix, quadtree, approximate, wide, all noise), device
and host path compared: python tools/path_smoke.py. Exits non-zero on an error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1912_06255_b200 as pkg  # noqa: E402

cases = [
    ("3d csr", datagen.seed_spreader(20_000, 3, 20_000, 1, 0.02, noise_frac=0.03), 200, 15, 0, None),
    ("7d brute", datagen.seed_spreader(10_000, 7, 30_000, 2, 0.02), 900, 20, 0, None),
    ("5d tree", datagen.seed_spreader(10_000, 5, 30_000, 3, 0.02), 600, 20, pkg.F_FORCE_TREE, None),
    ("3d sparse brick", datagen.uniform(60_000, 3, 40_000, 4), 500, 3, 0, None),
    ("3d sparse brick ovf", np.concatenate([datagen.uniform(60_000, 3, 40_000, 5),
                                            np.full((4000, 3), 777, np.int32)]), 500, 10, 0, None),
    ("3d sparse thread", datagen.uniform(60_000, 3, 40_000, 4), 500, 3, pkg.F_NO_BRICK, None),
    ("2d sparse", datagen.uniform(50_000, 2, 20_000, 6), 150, 6, 0, None),
    ("1d", datagen.uniform(20_000, 1, 200_000, 7), 3, 3, 0, None),
    ("radix", datagen.uniform(30_000, 3, 1_000_000, 8), 3000, 3, pkg.F_RADIX_GROUP, None),
    ("quadtree", datagen.seed_spreader(20_000, 3, 5_000, 9, 0.02), 300, 40, pkg.F_QUADTREE, None),
    ("approx", datagen.seed_spreader(20_000, 3, 20_000, 10, 0.02), 200, 15, 0, 0.5),
    ("wide", datagen.uniform(5_000, 3, 2_000_000_000, 11), 300_000_000, 4, pkg.F_FORCE_WIDE, None),
    ("all noise", datagen.uniform(50_000, 3, 100_000, 12), 500, 10_000, 0, None),
]
for name, pts, eps, mp, fl, rho in cases:
    t = torch.from_numpy(np.ascontiguousarray(pts, np.int32)).cuda()
    r = pkg.dbscan(t, eps, mp, flags=fl, rho=rho)
    torch.cuda.synchronize()
    h = pkg.dbscan(np.ascontiguousarray(pts, np.int32), eps, mp, flags=fl, rho=rho)
    assert np.array_equal(r.cluster.cpu().numpy(), h.cluster), name
    print(f"{name:22s} core {r.n_core:7d} clusters {r.n_clusters:6d} border {r.n_border:6d} "
          f"sparse {r.stats['sparse']} brick {r.stats['brick']}")
print("ok")
