#!/usr/bin/env python3
"""Assemble profiles/rN_traffic.json (read by bench.py) from ncu --set full raw
CSVs of tools/prof.sh, one per config: per-kernel DRAM bytes per launch, the
dominant MarkCore kernels, and the grouping stage's bytes per call (kernels
lat_*, group_*, hash_*, radix_*, segment*, sample_collisions; the shared
scan_kernel is left out since other stages launch it too).

usage: python tools/make_traffic.py c5_10=gpurun_out/a_raw.csv c3=... > profiles/r1_traffic.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_traffic import load  # noqa: E402

GROUP = ("lat_", "group_", "hash_", "radix", "segment", "sample_collisions")
out = {"note": "DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch from ncu --set full "
               "(cold L2: ncu flushes caches before each replay) on tools/run_one.py; "
               "see profiles/r1_ncu_*_table.txt", "grouping": {}, "kernels": {}}
for arg in sys.argv[1:]:
    run, path = arg.split("=", 1)
    k = load(path)
    out["kernels"][run] = k
    g = sum(v["dram_bytes_per_launch"] * v["launches"] for n, v in k.items() if n.startswith(GROUP))
    kind = "lattice" if any(n.startswith("lat_") for n in k) else "hash"
    out["grouping"][f"{run} ({kind})"] = g
    for name in ("sp_core_brick_kernel", "sp_core_kernel"):
        if name in k and name not in out:
            out[name] = k[name]["dram_bytes_per_launch"]
print(json.dumps(out, indent=1, sort_keys=True))
