#!/usr/bin/env python3
"""Assemble profiles/r2_traffic.json (read by bench.py) from ncu --set full raw
CSVs of tools/prof.sh (one call per run, every kernel): DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum) per call of each stage's
kernels, keyed {run: {stage: bytes}}, plus the per-kernel table. The shared
scan_kernel is left out (several stages launch it).

usage: python tools/make_traffic.py c5_10=gpurun_out/a_raw.csv c3=... > profiles/r2_traffic.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_traffic import load  # noqa: E402

STAGES = [  # (stage, kernel-name prefixes)
    ("a1 bbox", ("bbox", "sample_collisions")),
    ("a2-a3 grouping", ("lat_", "group_", "radix", "segment", "keys_kernel")),
    ("a4-a5 neighbour cells", ("nbr_", "hash_insert", "dense_fill", "tree_", "morton", "decode_cells", "bucket_",
                               "sort_rows")),
    ("a6 MarkCore", ("sp_core_brick", "sp_core_kernel", "mark_core", "qt_", "qb_")),
    ("a7 compaction", ("sp_cells", "partition", "core_count", "dir_set", "popc", "dir_pack", "core_list")),
    ("a8 ClusterCore", ("sp_pairs", "sp_core_pack", "wave_csr", "bcp_large", "uf_")),
    ("a9 labels", ("label_roots", "cell_label", "write_points", "write_positions", "core_from_cluster")),
    ("a10 ClusterBorder", ("sp_border", "border_")),
]
out = {"note": "DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per call of each stage's kernels, "
               "ncu --set full (cold L2: ncu flushes caches before each replay, an upper bound for inputs "
               "that are L2-resident in a real run) on tools/run_one.py; scan_kernel (shared) left out"}
kern = {}
for arg in sys.argv[1:]:
    run, path = arg.split("=", 1)
    k = load(path)
    kern[run] = k
    out[run] = {}
    for stage, pre in STAGES:
        b = sum(v["dram_bytes_per_launch"] * v["launches"] for n, v in k.items() if n.startswith(pre))
        if b:
            out[run][stage] = b
out["kernels"] = kern
print(json.dumps(out, indent=1, sort_keys=True))
