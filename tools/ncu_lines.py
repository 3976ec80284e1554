"""Stall samples per CUDA source line of one kernel (ncu source page, cuda view).
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [n]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"Line No"')][0]
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"File')), len(lines))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:end]))))
h = rows[0]
h[1] = "Source"
rows = [rows[0]] + [r for r in rows[1:] if r and r[0]]
si = h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed")
stalls = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
tot = sum(int(r[si] or 0) for r in rows[1:] if r[si].isdigit())
top = sorted((r for r in rows[1:] if r[si].isdigit()), key=lambda r: -int(r[si]))[:n]
for r in top:
    st = sorted(((int(r[i] or 0), h[i][6:]) for i in stalls if (r[i] or "0").isdigit()), reverse=True)[:3]
    s = " ".join(f"{k}:{v}" for v, k in st if v)
    print(f"{int(r[si])/max(tot,1):6.1%} L{r[0]:>4} exec={r[ei]:>9} [{s}] {r[1].strip()[:70]}")
