"""Per-phase timeline of the persistent K2 kernel (instrumented build).
usage: make trace && TSR_LIB=build/libtilesplat_b200_trace.so python tools/k2_trace.py [c2|c3]"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_19489_b200 as ts  # noqa: E402
from paper_2601_19489_b200 import _lib  # noqa: E402
from paper_2601_19489_b200.synthetic import make_scene  # noqa: E402

cfg = {"c2": (1_000_000, False), "c3": (3_000_000, True)}[sys.argv[1] if len(sys.argv) > 1 else "c2"]
params, cam, gt = make_scene(cfg[0], 1920, 1080, seed=0, clustered=cfg[1])
gset = ts.GaussianSet(**params)
camera = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 1920, 1080, cam["R"], cam["t"])
gt_dev = torch.from_numpy(np.asarray(gt, np.float32)).cuda()
st = ts.TrainStep(gset, ts.TrainConfig(max_iters=30_000), extent=4.0)
lib = _lib.load()
for _ in range(5):
    st.step(camera, gt_dev)
    torch.cuda.synchronize()
    if not hasattr(lib, "tsr_k2_trace_read"):  # plain build (e.g. under ncu)
        continue
    buf = (ctypes.c_ulonglong * 128)()
    lib.tsr_k2_trace_read(buf, None)
    t = np.array(buf[:33], dtype=np.int64)
    n = int(np.count_nonzero(t[1:]))
    print("K2 phase ends (us from start):", [round((x - t[0]) / 1e3, 1) for x in t[1:1 + n]])
    e = np.array(buf[40:48], dtype=np.int64)
    print("   emission CTA0 (gathers, scan, window-expand..., rewalk, end, expand, copy, kernel end):",
          [round((x - t[0]) / 1e3, 1) for x in e])
    for c in range(10):
        sub = np.array(buf[64 + 6 * c:70 + 6 * c], dtype=np.int64)
        if sub[0]:
            print(f"   scatter call {c} CTA0 first sub-tile (loads, rank, scan, stage, store, phase end):",
                  [round((x - t[0]) / 1e3, 1) for x in sub])
    # per-CTA arrival at each barrier (bar_base != NULL selects that buffer)
    if _ != 4:
        continue
    arr = (ctypes.c_ulonglong * (2048 * 32))()
    lib.tsr_k2_trace_read(arr, ctypes.c_void_p(1))
    a = np.array(arr, dtype=np.int64).reshape(2048, 32)
    g = int(np.count_nonzero(a[:, 0]))
    a = a[:g, :n]
    rel = (a - t[0]) / 1e3
    print(f"   arrivals over {g} CTAs: barrier: min / median / max (us) [slowest CTA]")
    for b in range(n):
        print(f"     b{b:2d}: {rel[:, b].min():7.1f} {np.median(rel[:, b]):7.1f} {rel[:, b].max():7.1f}"
              f" [{int(rel[:, b].argmax())}]")
