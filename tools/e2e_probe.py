#!/usr/bin/env python3
"""Timeline of the e2e leg: T host threads call the blocking host-buffer C ABI
on the bench suite (pinned buffers), K steps; prints every step's wall time and,
for the last step, each call's [start, end] in ms.
usage: python tools/e2e_probe.py [T] [K]"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1912_06255_b200 as pkg  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 3
K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
runs = ["c2", "c3", "c4_5d", "c4_7d", "c5_10", "c5_10k"]
host = []
for name in runs:
    cfg = datagen.CONFIGS[name]
    pts = torch.from_numpy(cfg.points()).pin_memory()
    outs = (torch.empty(cfg.n, dtype=torch.uint8).pin_memory(), torch.empty(cfg.n, dtype=torch.int32).pin_memory(),
            torch.empty(cfg.n + 1, dtype=torch.int64).pin_memory(), torch.empty(cfg.n, dtype=torch.int32).pin_memory())
    host.append((name, cfg, pts, outs))
ORD = os.environ.get("ORDER")
order = ([runs.index(x) for x in ORD.split(",")] if ORD
         else sorted(range(len(host)), key=lambda k: -host[k][2].numel()))
streams = [torch.cuda.Stream() for _ in range(T)]


def step():
    nxt, lock, log = [0], threading.Lock(), []
    t0 = time.perf_counter()

    def worker(w):
        torch.cuda.set_device(0)
        while True:
            with lock:
                if nxt[0] >= len(order):
                    return
                k = order[nxt[0]]
                nxt[0] += 1
            name, cfg, pts, outs = host[k]
            a = time.perf_counter()
            pkg.dbscan(pts, cfg.eps, cfg.min_pts, out=outs, stream=streams[w])
            log.append((name, w, (a - t0) * 1e3, (time.perf_counter() - t0) * 1e3))
    ths = [threading.Thread(target=worker, args=(w,)) for w in range(T)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    return (time.perf_counter() - t0) * 1e3, log


for i in range(K):
    ms, log = step()
    print(f"step {i}: {ms:.2f} ms  ({51e6 / ms * 1e3:.3g} points/s)")
for name, w, a, b in sorted(log, key=lambda x: x[2]):
    print(f"  {name:7s} thread {w}: {a:7.2f} .. {b:7.2f} ms")
