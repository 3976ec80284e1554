"""Summarise bench logs: python tools/benchsum.py gpurun_out/bench_*.log"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads([x for x in open(f) if x.startswith("{")][-1])
        ph = {k: round(v * 1e3, 1) for k, v in d["phases_ms"].items()}
        print(f"{f:40s} {d['ms_per_step']:.4f} ms  {ph}")
    except Exception:
        print(f"{f:40s} ERR {open(f).read()[-200:]!r}")
