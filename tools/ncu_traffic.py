#!/usr/bin/env python3
"""Per-kernel DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) and
duration from an ncu --set full raw CSV (tools/prof.sh NAME_raw.csv), as JSON.

usage: python tools/ncu_traffic.py gpurun_out/X_raw.csv [...]  > profiles/rN_traffic_X.json
Kernels launched several times in one capture get the mean per launch.
Note: ncu flushes caches before each replayed kernel (cold L2), so these
bytes are an upper bound for kernels whose inputs are L2-resident in a run.
"""
import collections
import csv
import json
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "msecond": 1e-3, "second": 1.0}


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    out = collections.defaultdict(list)
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").split("<")[0]
        name = name.replace("db::", "")

        def val(m):
            v = float(r[ix[m]].replace(",", ""))
            return v * UNITS.get(units[ix[m]], 1.0)
        out[name].append({"dram_bytes": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                          "duration_s": val("gpu__time_duration.sum")})
    return {k: {"dram_bytes_per_launch": sum(x["dram_bytes"] for x in v) / len(v),
                "ncu_duration_s": sum(x["duration_s"] for x in v) / len(v), "launches": len(v)}
            for k, v in out.items()}


if __name__ == "__main__":
    res = {}
    for p in sys.argv[1:]:
        res.update(load(p))
    print(json.dumps(res, indent=1, sort_keys=True))
