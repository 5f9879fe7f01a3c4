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
as it stands, on complete BASELINE runs (c2, c3, c4 5D and 7D: ~13 s of
O2 on 16 cores per step), timed on the host cores. It is a deliberately slow
reference.
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
# CPU baseline / reference arm sample: complete BASELINE runs (no prefixes:
# a prefix of walk-ordered seed-spreader data is another workload), the ones
# whose O2 time on all host cores fits the ~10-30 s budget (measured on the
# GPU box's 16 cores: 0.1 + 1.5 + 3.2 + 8.4 s). c5 (17-18 s per run with
# O2 on 16 cores) is timed in profiles/r2_cpu_baselines.jsonl with O1 and
# single-threaded O2 (tools/cpu_baselines.py).
REF_RUNS = ["c2", "c3", "c4_5d", "c4_7d"]
E2E_THREADS = int(os.environ.get("DB_E2E_THREADS", "3"))


# Stage rooflines. Algorithmic work per
# stage and run: HBM stages in bytes (SURVEY §8(d) formulas), distance-test
# stages in tests counted by the measurement build (libdbscan_b200_count.so,
# an untimed pass in a subprocess). Denominators: MEASURED_PEAKS.json hbm_gbs
# (driver-measured copy bandwidth) and U1 `peak_dist` (dbscan_peak_dist,
# measured live here: the shipped predicate on shared-memory tiles, best of
# 1/2/4 register queries per thread, at the run's d and arithmetic path).
STAGE_DEF = [  # (stage key in stage_ms, row, bound, kernels)
    ("bbox", "a1 bbox", "hbm", "bbox_kernel"),
    ("keys+sort", "a2-a3 grouping", "hbm", "group_count/group_scatter (hash), lat_* (lattice), keys+radix_pass"),
    ("segment", "a2-a3 grouping", "hbm", "segment_kernel (radix path)"),
    ("neighbors", "a4-a5 neighbour cells", "l2", "nbr_stencil / nbr_brute / tree_query"),
    ("markcore", "a6 MarkCore", "alu", "sp_core_brick_kernel / sp_core_kernel / mark_core_*"),
    ("compact", "a7 compaction", "hbm", "sp_cells_kernel / core_count_kernel / partition_kernel"),
    ("cluster", "a8 ClusterCore", "alu", "sp_pairs_kernel / wave_csr_kernel / bcp_large_kernel"),
    ("labels", "a9 labels", "hbm", "label_roots_kernel ... core_from_cluster_kernel"),
    ("border", "a10 ClusterBorder", "alu", "sp_border_emit_kernel / border_kernel + count/scan/fill"),
]


def stage_work(row, cfg, st, work):
    """Algorithmic work of one stage of one run: (amount, unit) — bytes for
    HBM stages, distance tests for the ALU stages."""
    n, d, nc = cfg.n, cfg.d, st["ncells"]
    if row == "a1 bbox":
        return 4 * d * n, "B"
    if row == "a2-a3 grouping":
        # read the points, write them grouped, the permutation and the cell
        # tables (SURVEY §8(d) minimum 2*4dn + 4n + 40 ncells); a run that
        # ended at Alg 2's global bound after the count pass read the points once
        return (2 * 4 * d * n + 4 * n + 40 * nc) if nc else 4 * d * n, "B"
    if row == "a7 compaction":
        return n + 8 * nc, "B"  # core flags read, core count + list per cell
    if row == "a9 labels":
        return 9 * n + 8 * nc, "B"  # n (1+4+4) + 8 ncells
    # MarkCore: the tests of Alg 2 as written (the cell-level
    # stencil walk, nearest column first, stopping at minPts) — the brick
    # kernel's sub-cell stencils run fewer (executed_tests, reported beside)
    key = {"a6 MarkCore": "markcore_alg2", "a8 ClusterCore": "bcp_tests", "a10 ClusterBorder": "border_tests"}.get(row)
    if key and work is not None:
        return work.get(key, work.get("markcore_tests", 0) if row == "a6 MarkCore" else 0), "tests"
    return None, None


def executed_tests(row, work):
    """Distance tests the kernels actually ran (measurement build)."""
    key = {"a6 MarkCore": "markcore_tests", "a8 ClusterCore": "bcp_tests", "a10 ClusterBorder": "border_tests"}.get(row)
    return work.get(key) if key and work else None


def measure_peaks(pkg, dims, wide_dims):
    """U1 peak_dist per (d, path): max over register tiles qt = 1, 2, 4."""
    out = {}
    for d in sorted(dims):
        # (variant 3: the brick MarkCore's predicate on packed rows, d = 3)
        for v in ([0] + ([1] if d in wide_dims else []) + ([3] if d == 3 else [])):
            best = max(pkg.peak_dist(d, v, qt, reps=60)["tests_per_s"] for qt in (1, 2, 4))
            out[(d, v)] = best
    return out


def load_traffic():
    """Per-launch DRAM bytes (read + write) from the committed ncu --set full
    summary (profiles/r2_traffic.json), or {} when absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as f:
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


# ------------------------------------------------------------ work pass
def work_pass_child(args):
    """(subprocess, DBSCAN_B200_COUNT=1) one call per run through the
    measurement build; prints {run: {markcore_tests, bcp_tests, border_tests}}."""
    import torch
    import paper_1912_06255_b200 as pkg
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    out = {}
    for name in [r for r in args.runs.split(",") if r]:
        cfg = datagen.CONFIGS[name]
        r = pkg.dbscan(torch.from_numpy(cfg.points()).to(dev), cfg.eps, cfg.min_pts)
        assert r.stats["counting_build"] == 1, "work pass: not the measurement build"
        out[name] = {k: r.stats[k] for k in ("markcore_tests", "markcore_alg2", "bcp_tests", "border_tests")}
        del r
    print("WORK " + json.dumps(out), flush=True)


def run_work_pass(runs, local):
    env = dict(os.environ, DBSCAN_B200_COUNT="1", LOCAL_RANK=str(local))
    for k in ("RANK", "WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.abspath(__file__), "--work-pass", "--runs", ",".join(runs)],
                       env=env, capture_output=True, text=True)
    for line in p.stdout.splitlines():
        if line.startswith("WORK "):
            return json.loads(line[5:])
    print("work pass failed:", p.stderr[-2000:], file=sys.stderr)
    return {}


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
    """Time the CPU oracle O2, as it stands, on complete BASELINE runs (REF_RUNS)
    on all host cores: each step is one O2 call per run."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    samples = []
    for name in REF_RUNS:
        cfg = datagen.CONFIGS[name]
        samples.append((name, np.ascontiguousarray(cfg.points()), cfg.eps, cfg.min_pts))
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
    sample = (f"O2 CPU grid oracle (OpenMP, {cores} threads) on the complete runs {','.join(REF_RUNS)} "
              f"({npts} points per step); c5 timed separately (profiles/r2_cpu_baselines.jsonl)")
    line = {"metric": METRIC, "value": value, "unit": "points/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * total / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": "suite: BASELINE configs[1..4] (c2,c3,c4_5d,c4_7d,c5 minPts 10 and 1e4)",
                       "runs": REF_RUNS, "sample": sample},
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
    ap.add_argument("--no-work", action="store_true", help="skip the work-counting pass (no ALU fractions)")
    ap.add_argument("--no-small", action="store_true", help="skip the configs[0] (c1) fixed-cost line")
    ap.add_argument("--work-pass", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.work_pass:
        return work_pass_child(args)

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

    # algorithmic work of the distance-test stages: the measurement build in a
    # subprocess (untimed; one call per run), and U1 peaks measured live
    work = {} if args.no_work else run_work_pass(runs, local)
    peaks_u1 = measure_peaks(pkg, {c.d for _, c, _, _ in data}, set())
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

    # ---- rooflines per run and stage
    peak, peak_kind = load_peaks()
    traffic = load_traffic()
    stage_tot = {}
    for i in range(len(runs)):
        for k, v in stage_acc[i].items():
            if k != "total":
                stage_tot[k] = stage_tot.get(k, 0.0) + v
    step_stage_ms = sum(stage_tot.values()) / args.steps
    rooflines = []
    for i, (name, cfg, t, _) in enumerate(data):
        st = stats[i]
        merged = {}
        for key, row, bound, kern in STAGE_DEF:
            ms = stage_acc[i].get(key, 0.0) / args.steps
            if ms <= 0:
                continue
            e = merged.setdefault(row, {"run": name, "stage": row, "bound": bound, "kernel": kern, "ms": 0.0})
            e["ms"] += ms
            if key == "segment":
                e["kernel"] += " + " + kern
        for row, e in merged.items():
            amount, unit = stage_work(row, cfg, st, work.get(name))
            e["ms_share"] = e["ms"] / max(1e-9, step_stage_ms)
            e["ms"] = round(e["ms"], 4)
            if amount is None or e["bound"] == "l2":
                e["frac"] = None
                rooflines.append(e)
                continue
            if unit == "B":
                ach = amount / (e["ms"] / 1e3) / 1e9
                e.update({"achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                          "algorithmic": amount, "peak_kind": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"})
            else:
                # the predicate the stage's kernel ran: the brick MarkCore's
                # packed-row test, else the shipped uint32 / 64-bit one
                brick = row == "a6 MarkCore" and st.get("brick", 0) >= 1
                pk = peaks_u1.get((cfg.d, 3)) if brick else peaks_u1.get((cfg.d, 1 if st["wide"] else 0))
                if not amount or not pk:
                    e["frac"] = None
                    rooflines.append(e)
                    continue
                ach = amount / (e["ms"] / 1e3)
                ex = executed_tests(row, work.get(name))
                if ex is not None and ex != amount:
                    e.update({"executed_tests": ex, "executed_frac": ex / (e["ms"] / 1e3) / pk})
                e.update({"achieved": ach / 1e12, "peak": pk / 1e12, "unit": "T distance tests/s",
                          "frac": ach / pk, "algorithmic": amount,
                          "peak_kind": f"U1 peak_dist measured live (d={cfg.d}, "
                                       f"{'brick packed-row' if brick else ('64-bit' if st['wide'] else 'uint32')} predicate)"})
            e["traffic"] = traffic.get(name, {}).get(row)
            rooflines.append(e)
    # the headline: the stage with the largest share of the step (a single
    # kernel dominates it: c5's MarkCore brick kernel, one launch per run)
    cand = [r for r in rooflines if r.get("frac") is not None]
    roofline = None
    if cand:
        top = max(cand, key=lambda r: r["ms_share"])
        roofline = {k: top.get(k) for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")}
        if "executed_tests" in top:
            roofline.update({"executed_tests_per_launch": top["executed_tests"], "executed_frac": top["executed_frac"],
                             "algorithmic_note": "Alg 2's tests (P:L571-598, cell-level stencil walk stopping at "
                                                 "minPts, counted by the measurement build); the kernel's sub-cell "
                                                 "stencils skip candidates no point of the sub-cell can reach "
                                                 "(executed_tests, executed_frac)"})
        roofline.update({"run": top["run"], "stage": top["stage"], "kernel": top["kernel"],
                         "ms_per_launch": top["ms"], "ms_share": top["ms_share"],
                         "algorithmic_per_launch": top["algorithmic"], "peak_kind": top["peak_kind"],
                         "traffic_note": "DRAM bytes (read + write) of the stage's kernels per call, ncu --set full "
                                         "(cold L2), profiles/r2_traffic.json (current build; r2a_traffic.json: the earlier round-2 build)"})
    peaks_out = {f"d{d}_{ {0: 'u32', 1: 'i64', 3: 'brick'}[v] }": round(p / 1e12, 4) for (d, v), p in peaks_u1.items()}

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

    # ---- CPU baseline: the oracle as it stands, bounded sample (rank 0, N=1):
    # O2 on all host cores over the complete runs REF_RUNS
    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        import oracle
        oracle.build()
        t0 = time.perf_counter()
        npts = 0
        for name, cfg, _, pts in data:
            if name in REF_RUNS:
                oracle.o2(np.ascontiguousarray(pts), cfg.eps, cfg.min_pts)
                npts += cfg.n
        dt = time.perf_counter() - t0
        if npts:
            cpu = {"value": npts / dt, "unit": "points/s", "cores": os.cpu_count(), "kind": "oracle",
                   "sample": f"O2 CPU grid oracle (OpenMP, {os.cpu_count()} threads) on the complete runs "
                             f"{','.join(r for r in REF_RUNS if r in runs)} ({npts} points, {dt:.1f} s); c5 runs "
                             "timed in profiles/r2_cpu_baselines.jsonl (O2 16 threads: 17-18 s each)"}

    # ---- configs[0] (c1, 10K points): not part of the 10M-point metric; its
    # per-call time (fixed cost: launches and synchronisations) reported beside it
    small = None
    if rank == 0 and not args.no_small:
        cfg = datagen.CONFIGS["c1"]
        t1 = torch.from_numpy(cfg.points()).to(dev)
        ms1 = []
        for it in range(25):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pkg.dbscan(t1, cfg.eps, cfg.min_pts)
            e1.record(stream)
            e1.synchronize()
            if it >= 5:
                ms1.append(e0.elapsed_time(e1))
        m1 = statistics.median(ms1)
        small = {"run": "c1", "n": cfg.n, "ms_median": round(m1, 4), "pts_per_s": cfg.n / (m1 / 1e3),
                 "note": "configs[0], 10K points: per-call fixed cost (device time, CUDA events, median of 20)"}

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
            "roofline": roofline, "rooflines": rooflines, "u1_peak_T_tests_per_s": peaks_out, "stage_ms_per_step": {k: round(v / args.steps, 4) for k, v in stage_tot.items()},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "small_config": small,
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
