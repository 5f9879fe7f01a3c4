#!/bin/bash
# Per-launch device times of one config run through the C ABI (the last of
# REPS calls), in launch order, as text: tools/seq.sh NAME CONFIG [REPS] [FLAGS]
set -u
name=$1; cfg=$2; reps=${3:-2}; flags=${4:-0}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "/tmp/${name}.csv" \
    python tools/run_one.py "$cfg" "$reps" "$flags" > "gpurun_out/${name}_ncu.log" 2>&1
python - "$name" "$reps" <<'PY'
import csv, sys
name, reps = sys.argv[1], int(sys.argv[2])
rows = [r for r in csv.DictReader(l for l in open(f"/tmp/{name}.csv") if not l.startswith("=="))]
ks = []
for r in rows:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        v = float(r["Metric Value"]); u = r["Metric Unit"]
        v = v / 1000 if u in ("ns", "nsecond") else (v * 1000 if u in ("ms", "msecond") else v)
        ks.append((r["ID"], r["Kernel Name"][:70], v))
per = len(ks) // reps
last = ks[-per:] if per else ks
with open(f"gpurun_out/{name}_seq.txt", "w") as f:
    tot = sum(v for _, _, v in last)
    for i, (_, k, v) in enumerate(last):
        f.write(f"{i:3d} {v:9.1f} us  {k}\n")
    f.write(f"total {tot:.1f} us over {len(last)} launches\n")
PY
