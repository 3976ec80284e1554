"""Per-kernel key metrics of an ncu --set full report as JSON (first launch of each kernel).
usage: python tools/ncu_summary.py report.ncu-rep > profiles/<name>.json"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "lts__t_sector_hit_rate.pct"]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
units = rows[1]
seen, res = set(), []
for r in rows[2:]:
    k = r[h.index("Kernel Name")]
    if k in seen:
        continue
    seen.add(k)
    d = {"Kernel Name": k}
    u = {}
    for m in METRICS:
        if m in h:
            d[m] = r[h.index(m)]
            u[m] = units[h.index(m)]
    d["units"] = u
    res.append(d)
json.dump(res, sys.stdout, indent=1)
