#!/usr/bin/env python3
"""Run one BASELINE config through the C ABI a few times (for ncu / sanitizer
captures). Usage: python tools/run_one.py c3 [reps] [flags]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1912_06255_b200 as pkg  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = datagen.CONFIGS[name]
t = torch.from_numpy(cfg.points()).cuda()
for i in range(reps):
    r = pkg.dbscan(t, cfg.eps, cfg.min_pts, flags=flags, timing=True)
    torch.cuda.synchronize()
print(name, r.n_core, r.n_clusters, r.n_border, r.stats, {k: round(v, 3) for k, v in r.stage_ms.items()})
