import sys, time
sys.path.insert(0, ".")
import torch, numpy as np, ctypes as C
import datagen, paper_1912_06255_b200 as pkg
pts = torch.from_numpy(datagen.seed_spreader(20_000, 3, 1e6, 1, 0.01)).cuda()
dev = pts.device
def tm(f, n=2000):
    f()
    t = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t) / n * 1e6
print("empty x3", tm(lambda: (torch.empty(20000, dtype=torch.uint8, device=dev), torch.empty(20000, dtype=torch.int32, device=dev), torch.empty(20001, dtype=torch.int64, device=dev))))
print("current_stream", tm(lambda: torch.cuda.current_stream(dev)))
def ctx():
    with torch.cuda.device(dev):
        pass
print("device ctx", tm(ctx))
print("contiguous", tm(lambda: pts.contiguous()))
print("Result()", tm(lambda: pkg._Result()))
r = pkg.dbscan(pts, 1000, 100)
torch.cuda.synchronize()
def call():
    pkg.dbscan(pts, 1000, 100)
t = time.perf_counter()
for _ in range(50): call()
torch.cuda.synchronize()
print("full call (host, incl. GPU)", (time.perf_counter() - t) / 50 * 1e6)
