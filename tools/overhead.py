#!/usr/bin/env python3
"""Fixed per-call cost: device time of dbscan() on small inputs of each path
(CUDA events around the call, median of 20), with the library's stage times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1912_06255_b200 as pkg  # noqa: E402

cases = [("c1", datagen.CONFIGS["c1"].points(), 5000, 10),
         ("3d-csr", datagen.seed_spreader(20_000, 3, 1e6, 1, 0.01), 1000, 100),
         ("7d-csr", datagen.seed_spreader(20_000, 7, 1e5, 2, 0.01), 2000, 100),
         ("3d-sparse", datagen.uniform(20_000, 3, 30_000, 3), 500, 10),
         ("3d-noise", datagen.uniform(20_000, 3, 30_000, 3), 500, 10_000)]
for name, pts, eps, mp in cases:
    t = torch.from_numpy(np.ascontiguousarray(pts, np.int32)).cuda()
    ms = []
    for it in range(25):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = pkg.dbscan(t, eps, mp)
        e1.record()
        e1.synchronize()
        if it >= 5:
            ms.append(e0.elapsed_time(e1))
    r = pkg.dbscan(t, eps, mp, timing=True)
    torch.cuda.synchronize()
    st = {k: round(v * 1e3) for k, v in r.stage_ms.items()}
    print(f"{name:10s} {np.median(ms) * 1e3:7.0f} us  launches {r.stats['launches']:3d}  stages(us) {st}")
