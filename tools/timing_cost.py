import sys; sys.path.insert(0, ".")
import torch, statistics, datagen, paper_1912_06255_b200 as pkg
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
for name in ["c2", "c3", "c4_7d", "c5_10", "c5_10k"]:
    cfg = datagen.CONFIGS[name]
    t = torch.from_numpy(cfg.points()).cuda()
    res = {}
    for timing in (True, False, True, False):
        ms = []
        for _ in range(8):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            r = pkg.dbscan(t, cfg.eps, cfg.min_pts, timing=timing)
            e1.record(st)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        res.setdefault(timing, []).append(statistics.median(ms[2:]))
    print(name, {k: [round(x, 4) for x in v] for k, v in res.items()})
