#!/usr/bin/env python3
"""BASELINE.md §5 table from a bench.py JSON line and the CPU-baseline lines of
tools/cpu_baselines.py. usage: python tools/baseline_table.py bench.json cpu.jsonl"""
import json
import sys


def main():
    b = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    cpu = [json.loads(l) for l in open(sys.argv[2]) if l.strip()]
    host = next((c["host"] for c in cpu if "host" in c), {})
    o1 = {(c["run"], c["threads"]): c["seconds"] for c in cpu if c.get("oracle") == "O1"}
    o2 = {(c["run"], c["threads"]): c["seconds"] for c in cpu if c.get("oracle") == "O2"}
    nproc = host.get("nproc", 16)
    rows = {r["run"]: r for r in b["runs"]}
    roof = {}
    for e in b["rooflines"]:
        roof.setdefault(e["run"], {})[e["stage"]] = e
    print("| Run | GPU ms (median) | Mpts/s | Grouping GB/s (frac of 6.54 TB/s) | a6 MarkCore T tests/s (frac of U1) "
          "| a8 ClusterCore T tests/s (frac) | O1 s (threads) | O2 s, 1 thread / %d threads | Parity vs oracle |" % nproc)
    print("|---|---|---|---|---|---|---|---|---|")
    names = [("c1", "c1"), ("c2", "c2"), ("c3", "c3"), ("c4_5d", "c4-5D"), ("c4_7d", "c4-7D"),
             ("c5_10", "c5, minPts 10"), ("c5_10k", "c5, minPts 10⁴")]
    small = b.get("small_config") or {}
    for key, label in names:
        if key == "c1":
            ms = small.get("ms_median")
            mpts = small.get("pts_per_s", 0) / 1e6 if small else None
            rf = {}
        else:
            r = rows.get(key, {})
            ms = r.get("ms_median")
            mpts = r.get("pts_per_s", 0) / 1e6 if r else None
            rf = roof.get(key, {})
        g = rf.get("a2-a3 grouping")
        a6 = rf.get("a6 MarkCore")
        a8 = rf.get("a8 ClusterCore")
        fmt = lambda e, u: (f"{e['achieved']:.{2 if u == 'GB/s' else 3}f} ({e['frac']:.3f})" if e and e.get("frac") is not None else "—")
        o1s = [f"{o1[(key, t)]:.2f} ({t})" for t in (1, nproc) if (key, t) in o1]
        o2s = " / ".join(f"{o2[(key, t)]:.2f}" for t in (1, nproc) if (key, t) in o2)
        parity = "bit-exact vs O1 (test_c1_full_vs_o1)" if key == "c1" else (
            "bit-exact vs O2 (test_c2_full_vs_o2)" if key == "c2" else
            "bit-exact vs O2 + 256 sampled O1 points (test_full_config, test_e2e_host_path_full)")
        print(f"| {label} | {ms if ms is not None else '—'} | {mpts:.0f} | {fmt(g, 'GB/s')} | {fmt(a6, 'T')} | "
              f"{fmt(a8, 'T')} | {', '.join(o1s) or '—'} | {o2s or '—'} | {parity} |"
              if mpts is not None else f"| {label} | — | — | — | — | — | {', '.join(o1s) or '—'} | {o2s or '—'} | {parity} |")
    print()
    print(f"Host: {host.get('lscpu_model', '?')}, nproc {nproc}. Bench: value {b['value']:.4g} points/s, "
          f"{b['ms_per_step']:.3f} ms per step, clocks {b.get('clocks', {}).get('sm_mhz')} MHz, "
          f"reasons {b.get('clocks', {}).get('reasons')}.")


if __name__ == "__main__":
    main()
