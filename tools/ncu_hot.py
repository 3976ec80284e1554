"""Top stall lines of one kernel's SASS source page from an ncu report.
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [n]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
# first kernel block only
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"')),
           len(lines))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:end]))))
h = rows[0]
si, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(int(r[si] or 0) for r in rows[1:])
top = sorted(rows[1:], key=lambda r: -int(r[si] or 0))[:n]
for r in top:
    print(f"{int(r[si])/max(tot,1):6.1%}  exec={r[ei]:>9}  {r[1].strip()[:90]}")
