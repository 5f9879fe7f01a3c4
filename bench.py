#!/usr/bin/env python3
"""bench.py — end-to-end exact grid DBSCAN throughput on B200.

Workload ("suite"): BASELINE.json configs[1..4] at full size — c2 (2D, 1M),
c3 (3D, 10M), c4 5D and 7D (10M each), c5 3D uniform at minPts 10 and 10^4
(10M each): 51M points per step over d = 2..7, the configurations the metric
"points/sec end-to-end exact grid DBSCAN (10M pts, d=2-7)" is quoted on.
configs[0] (10K points) is the oracle-sized parity case, not a bench line.

One step = one dbscan() call per run, i.e. the whole hot path (SURVEY §8
a1-a10) over every run's input. value = points processed / device time,
inputs resident in HBM, outputs allocated by the call; L2 is flushed (256 MB
write) before every run, outside the timed region. e2e = the same metric
through the C ABI with pinned HOST buffers, H2D of the points and D2H of all
outputs inside the timed region.

Multi-GPU (torchrun): the method runs on one GPU (BASELINE north_star); each
rank runs an independent replica of the suite ("replicas only", DESIGN.md
§Multi-GPU), value = points of all ranks / max-over-ranks device time.

--impl reference: the CPU oracle O2 (oracle/, the "simple CPU grid version")
as it stands, on a bounded sample of the same runs (a 5% prefix of each run's
points), timed on the host cores. It is a deliberately slow reference.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import datagen  # noqa: E402

METRIC = "points/sec end-to-end exact grid DBSCAN (10M pts, d=2–7); per-stage HBM GB/s"
SUITE = ["c2", "c3", "c4_5d", "c4_7d", "c5_10", "c5_10k"]
REF_FRACTION = 0.05
E2E_THREADS = int(os.environ.get("DB_E2E_THREADS", "3"))


# int32 issue peak: 148 SMs x 4 schedulers x 32 lanes x 1.965 GHz = 37.2 T
# lane-instructions/s; a 3D distance test is ~10 int32 SASS instructions
# (3 x VABSDIFF/VIMNMX/IMAD + compare): ~3.7e12 tests/s
INT_TESTS_PEAK = 148 * 4 * 32 * 1.965e9 / 10


def load_traffic():
    """Per-launch DRAM bytes (read + write) from the committed ncu --set full
    summary (profiles/r1_traffic.json), or {} when absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons sampled every 10 ms through NVML (the
    same counters nvidia-smi reads) on a thread, DURING the timed region."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.run = False
        self.err = None

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.run = True
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _loop(self):
        nv = self.nv
        while self.run:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, rs))
            except Exception as e:  # pragma: no cover
                self.err = str(e)
                return
            time.sleep(0.01)

    def stop(self):
        self.run = False
        if self.err and not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable: {self.err}"]}
        self.t.join(timeout=2)
        nv = self.nv
        reasons = sorted({name for _, rs in self.rows for name, attr in self.REASONS
                          if rs & getattr(nv, attr, 0)})
        sm = [r[0] for r in self.rows]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_sm,
                "reasons": reasons, "samples": len(self.rows), "source": "NVML, 10 ms"}


def job_value(npts_per_rank_step: int, steps: int, local_ms: float, dist=None, device="cpu"):
    """Whole-job throughput of N replicas ("replicas only"):
    points of all ranks / the slowest rank's device time (max over ranks).
    Returns (value, max_ms). dist: torch.distributed (initialised) or None."""
    world = 1
    if dist is not None:
        import torch
        world = dist.get_world_size()
        t = torch.tensor([local_ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        local_ms = float(t.item())
    return npts_per_rank_step * steps * world / (local_ms / 1000.0), local_ms


# --------------------------------------------------------------- e2e calls
def e2e_calls(pkg, host, order, streams, dev, keep=False):
    """One e2e step: len(streams) host threads, one CUDA stream each, take the
    runs from a shared queue (in `order`) and call the blocking host-buffer C
    ABI (pinned input, pinned caller-owned outputs). host[k] = (cfg, pinned
    points, (core, cluster, border_off, border_ids) pinned buffers).
    Returns (seconds, H2D bytes, D2H bytes, results by run if keep)."""
    import torch
    nthreads = len(streams)
    b_in = [0] * nthreads
    b_out = [0] * nthreads
    errs = []
    results = [None] * len(host)
    nxt = [0]
    lock = threading.Lock()

    def worker(w):
        try:
            torch.cuda.set_device(dev)
            while True:
                with lock:  # runs taken in turn from a shared queue
                    if nxt[0] >= len(order):
                        return
                    k = order[nxt[0]]
                    nxt[0] += 1
                cfg, hp, outs = host[k]
                r = pkg.dbscan(hp, cfg.eps, cfg.min_pts, out=outs, stream=streams[w])
                b_in[w] += hp.numel() * 4
                # bytes that cross the link: the library writes constant
                # outputs on the host (border_off when no point is a border
                # point; every output when no point is core)
                nnz = len(r.border_ids)
                if r.n_core:
                    b_out[w] += cfg.n * (1 + 4) + ((8 * (cfg.n + 1) + 4 * nnz) if nnz else 0)
                if keep:
                    results[k] = r
        except Exception as e:  # pragma: no cover
            errs.append(e)
    t0 = time.perf_counter()
    ths = [threading.Thread(target=worker, args=(w,)) for w in range(nthreads)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    dt = time.perf_counter() - t0
    if errs:
        raise errs[0]
    return dt, sum(b_in), sum(b_out), results


def e2e_order(host, dev_ms):
    """The run with the longest device time first (its kernels overlap the
    other runs' input copies), then by input size, largest first (measured on
    B200: 22.1 ms per step against 24.4 ms for input size alone)."""
    first = max(range(len(host)), key=lambda k: dev_ms[k])
    return [first] + sorted((k for k in range(len(host)) if k != first), key=lambda k: -host[k][1].numel())


def e2e_host_buffers(data, torch):
    """Pinned host input and caller-owned pinned output buffers per run."""
    host = []
    for name, cfg, _, pts in data:
        hp = torch.from_numpy(pts).pin_memory()
        outs = (torch.empty(cfg.n, dtype=torch.uint8).pin_memory(),
                torch.empty(cfg.n, dtype=torch.int32).pin_memory(),
                torch.empty(cfg.n + 1, dtype=torch.int64).pin_memory(),
                torch.empty(cfg.n, dtype=torch.int32).pin_memory())
        host.append((cfg, hp, outs))
    return host


# ------------------------------------------------------------- reference
def run_reference(args):
    """Time the CPU oracle O2 on a bounded sample of every run."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    samples = []
    for name in SUITE:
        cfg = datagen.CONFIGS[name]
        pts = cfg.points()
        k = max(1, int(len(pts) * REF_FRACTION))
        samples.append((name, np.ascontiguousarray(pts[:k]), cfg.eps, cfg.min_pts))
    oracle.build()
    times = []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        for _, p, e, m in samples:
            oracle.o2(p, e, m)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    npts = sum(len(s[1]) for s in samples)
    total = sum(times)
    value = npts * len(times) / total
    cores = os.cpu_count()
    sample = f"O2 CPU grid oracle on the first {REF_FRACTION:.0%} of each run's points ({npts} points/step)"
    line = {"metric": METRIC, "value": value, "unit": "points/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * total / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": "suite: BASELINE configs[1..4] (c2,c3,c4_5d,c4_7d,c5 minPts 10 and 1e4)",
                       "runs": SUITE, "sample": sample},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--runs", default=",".join(SUITE), help="comma list of runs (default: the suite)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--detail", action="store_true", help="print per-run stage times to stderr")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import paper_1912_06255_b200 as pkg
    pkg.load()

    runs = [r for r in args.runs.split(",") if r]
    data = []
    for name in runs:
        cfg = datagen.CONFIGS[name]
        pts = cfg.points()
        data.append((name, cfg, torch.from_numpy(pts).to(dev), pts))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def one_step(timing):
        ms, stages, launches, stats = [], [], 0, []
        for name, cfg, t, _ in data:
            flush.fill_(rank + 1)  # evict the inputs from L2 (outside the timed region)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = pkg.dbscan(t, cfg.eps, cfg.min_pts, timing=timing)
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
            stages.append(r.stage_ms)
            stats.append(r.stats | {"n_core": r.n_core, "n_clusters": r.n_clusters, "n_border": r.n_border,
                                    "nnz": int(r.border_ids.numel())})
            launches += r.stats["launches"]
            del r
        return ms, stages, launches, stats

    # algorithmic work of the sparse MarkCore: one counting run per run (untimed)
    work_tests = {}
    for name, cfg, t, _ in data:
        r = pkg.dbscan(t, cfg.eps, cfg.min_pts, flags=pkg.F_COUNT_WORK)
        if r.stats.get("markcore_tests"):
            work_tests[name] = r.stats["markcore_tests"]
        del r
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        one_step(True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    per_run_ms = [[] for _ in runs]
    stage_acc = [dict() for _ in runs]
    launches = 0
    stats = None
    for _ in range(args.steps):
        # the calls as a user makes them: no stage events (F_TIMING costs
        # 30-65 us of host work per call, after the kernels: measured)
        ms, _, l, stats = one_step(False)
        launches += l
        for i, m in enumerate(ms):
            per_run_ms[i].append(m)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = clk.stop()
    # stage times (rooflines, stage_ms): the same steps again with the
    # library's per-stage CUDA events, outside the timed region
    for _ in range(args.steps):
        _, stages, _, _ = one_step(True)
        for i in range(len(runs)):
            for k, v in stages[i].items():
                stage_acc[i][k] = stage_acc[i].get(k, 0.0) + v
    torch.cuda.synchronize()
    step_ms = [sum(per_run_ms[i][s] for i in range(len(runs))) for s in range(args.steps)]
    npts_step = sum(c.n for _, c, _, _ in data)
    value, total_ms = job_value(npts_step, args.steps, sum(step_ms), dist, dev)

    # ---- rooflines. Stage times come from CUDA events the
    # library records on the launching stream (F_TIMING); algorithmic work per
    # run from the run's shape and, for the sparse MarkCore, from one counting
    # run (F_COUNT_WORK) outside the timed region.
    peak, peak_kind = load_peaks()
    traffic = load_traffic()
    stage_tot = {}
    for i in range(len(runs)):
        for k, v in stage_acc[i].items():
            if k != "total":
                stage_tot[k] = stage_tot.get(k, 0.0) + v
    rooflines = []
    # grouping (a2-a4): the largest HBM stage; algorithmic bytes = read the
    # points twice + write the padded sorted points, index and cell id, plus
    # the cell table (12 B per cell); the radix path adds its key passes
    g_bytes = g_ms = 0.0
    for i, (name, cfg, t, _) in enumerate(data):
        st = stats[i]
        D = 2 if cfg.d <= 2 else (4 if cfg.d <= 4 else 8)
        by = (8 * cfg.d + 4 * D + 8) * cfg.n + 12 * st["ncells"]
        if st["hash_group"] == 0 and st["sort_passes"]:
            kb = 8 if st["key_bits"] > 32 else 4
            by += (kb + 4) * cfg.n + st["sort_passes"] * 2 * (kb + 4) * cfg.n
        g_bytes += by * args.steps
        g_ms += stage_acc[i].get("keys+sort", 0.0) + stage_acc[i].get("segment", 0.0)
    if g_ms > 0:
        ach = g_bytes / (g_ms / 1e3) / 1e9
        rooflines.append({"stage": "a2-a4 grouping", "bound": "hbm",
                          "kernel": "group_count/group_scatter (hash), lat_* (lattice), radix_pass+segment",
                          "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                          "traffic": traffic.get("grouping"),
                          "traffic_note": "DRAM bytes per call of the grouping kernels by run, ncu --set full (cold L2)",
                          "peak_kind": peak_kind,
                          "ms_share": g_ms / max(1e-9, sum(stage_tot.values())),
                          "note": "algorithmic bytes: 8d+4D+8 per point + 12 per cell (+ key passes on the radix path)"})
    # sparse MarkCore (a6): int32 ALU issue bound; tests per second
    for i, (name, cfg, t, _) in enumerate(data):
        if stats[i]["sparse"] and work_tests.get(name):
            ms = stage_acc[i].get("markcore", 0.0) / args.steps
            if ms <= 0:
                continue
            ach = work_tests[name] / (ms / 1e3) / 1e12
            tp = INT_TESTS_PEAK / 1e12
            kname = "sp_core_brick_kernel" if stats[i].get("brick") else "sp_core_kernel"
            rooflines.append({"stage": f"a6 MarkCore ({name})", "bound": "alu", "kernel": kname,
                              "achieved": ach, "peak": tp, "unit": "T distance tests/s", "frac": ach / tp,
                              "traffic": traffic.get(kname),
                              "traffic_note": "DRAM bytes per launch, ncu --set full (cold L2)",
                              "peak_kind": "derived (DESIGN.md §8): int32 issue rate / 10 SASS per 3D test",
                              "launch_ms": ms,
                              "ms_share": ms * args.steps / max(1e-9, sum(stage_tot.values())),
                              "tests_per_launch": work_tests[name]})
    # the headline is the dominant single KERNEL (the sparse MarkCore's
    # brick kernel, one launch per c5 run, the longest kernel of the step);
    # the grouping stage (several kernels per run) is reported beside it
    kern = [r for r in rooflines if r["bound"] == "alu"]
    roofline = max(kern or rooflines, key=lambda r: r["ms_share"]) if rooflines else None

    # ---- e2e through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        host = e2e_host_buffers(data, torch)
        h2d = d2h = 0
        streams = [torch.cuda.Stream(dev) for _ in range(E2E_THREADS)]
        dev_ms = [statistics.median(per_run_ms[k]) for k in range(len(host))]
        order = e2e_order(host, dev_ms)

        def e2e_step():
            nonlocal h2d, d2h
            dt, h2d, d2h, _ = e2e_calls(pkg, host, order, streams, dev)
            return dt
        # (at least 5: the first steps create and grow the threads' workspaces,
        # device memory mapped in the pool and pinned staging, ~0.2 s each)
        for _ in range(max(5, args.warmup)):
            w = e2e_step()
            if os.environ.get("DB_E2E_DEBUG"):
                print("e2e warm-up step ms:", round(w * 1e3, 2), file=sys.stderr)
        ts = [e2e_step() for _ in range(max(1, min(args.steps, 5)))]
        if os.environ.get("DB_E2E_DEBUG"):
            print("e2e step seconds:", [round(t * 1e3, 2) for t in ts], file=sys.stderr)
        e2e = {"value": npts_step * len(ts) / sum(ts), "unit": "points/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h,
               "timer": f"host wall clock around the step: {E2E_THREADS} host threads with one CUDA stream each take the runs from a shared queue and "
                        "call the blocking host-buffer C ABI (pinned inputs and outputs; the library copies inputs in turn)"}

    # ---- CPU baseline: the oracle as it stands, bounded sample (rank 0, N=1)
    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        import oracle
        oracle.build()
        t0 = time.perf_counter()
        npts = 0
        for name, cfg, _, pts in data:
            k = max(1, int(cfg.n * REF_FRACTION))
            oracle.o2(np.ascontiguousarray(pts[:k]), cfg.eps, cfg.min_pts)
            npts += k
        dt = time.perf_counter() - t0
        cpu = {"value": npts / dt, "unit": "points/s", "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"O2 CPU grid oracle on the first {REF_FRACTION:.0%} of each run's points "
                         f"({npts} points, {dt:.1f} s)"}

    run_info = []
    for i, (name, cfg, _, _) in enumerate(data):
        m = statistics.median(per_run_ms[i])
        run_info.append({"run": name, "n": cfg.n, "d": cfg.d, "eps": cfg.eps, "min_pts": cfg.min_pts,
                         "ms_median": round(m, 4), "pts_per_s": cfg.n / (m / 1000.0),
                         "stage_ms": {k: round(v / args.steps, 4) for k, v in stage_acc[i].items()},
                         "stats": stats[i]})
    line = {"metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": "suite: BASELINE configs[1..4] (c2,c3,c4_5d,c4_7d,c5 minPts 10 and 1e4)",
                       "runs": runs, "points_per_step": npts_step, "l2": "flushed (256 MB write) before every run",
                       "stage_timing": "stage_ms and rooflines from a second pass of the same steps with the library stage events (F_TIMING), outside the timed region",
                       "parallelism": "replicas" if world > 1 else "single GPU"},
            "roofline": roofline, "rooflines": rooflines, "stage_ms_per_step": {k: round(v / args.steps, 4) for k, v in stage_tot.items()},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "runs": run_info}
    if args.detail and rank == 0:
        for ri in run_info:
            print(ri["run"], ri["ms_median"], ri["stage_ms"], file=sys.stderr)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
