"""roofline.traffic for bench.py: DRAM bytes of ONE K4 (render_bwd) launch
from an `ncu --set full` capture.
usage: python tools/k4_traffic.py report.ncu-rep profiles/<summary>.json > profiles/k4_traffic.json
(the second argument names the committed per-kernel summary of the same capture)."""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
for r in rows[2:]:
    if "render_bwd" not in r[h.index("Kernel Name")]:
        continue
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        tot += float(r[h.index(m)]) * SCALE[units[h.index(m)]]
    t = float(r[h.index("gpu__time_duration.sum")])
    json.dump({"kernel": r[h.index("Kernel Name")], "bytes_per_launch": tot,
               "gpu_time_duration": t, "time_unit": units[h.index("gpu__time_duration.sum")],
               "source": f"dram__bytes_read.sum + dram__bytes_write.sum, first render_bwd launch "
                         f"of {sys.argv[1].split('/')[-1]} (summary: {sys.argv[2]})"},
              sys.stdout, indent=1)
    break
