#!/usr/bin/env python3
"""Per-kernel table from an .ncu-rep (needs ncu on PATH). Usage:
python tools/ncu_table.py report.ncu-rep"""
import csv
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__warps_active.avg.pct_of_peak_sustained_active",
     "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
ix = {h: i for i, h in enumerate(hdr)}
short = ["time", "dram_rd", "dram_wr", "sm%", "mem%", "occ%", "simt", "regs"]
print(f"{'kernel':34s} " + " ".join(f"{s:>12s}" for s in short))
for r in rows[2:]:
    vals = []
    for m in M:
        if m not in ix:
            vals.append("-")
            continue
        v, u = r[ix[m]], units[ix[m]]
        try:
            x = float(v.replace(",", ""))
            if u in ("byte", "Kbyte", "Mbyte", "Gbyte"):
                x *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}[u]
                vals.append(f"{x:10.1f}MB")
            elif u in ("nsecond", "usecond", "msecond"):
                x *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}[u]
                vals.append(f"{x:10.1f}us")
            else:
                vals.append(f"{x:12.1f}")
        except ValueError:
            vals.append(v[:12])
    print(f"{r[ix['Kernel Name']][:34]:34s} " + " ".join(f"{v:>12s}" for v in vals))
