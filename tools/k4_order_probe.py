"""K4r with its work units in K3's queue order vs longest-first (LPT, spans
computed on the host from the region list offsets) on the same C2 step's
buffers: device time of the K4r launch alone."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_19489_b200 as ts  # noqa: E402
from paper_2601_19489_b200.backward import backward_regions_raw  # noqa: E402
from paper_2601_19489_b200.synthetic import make_scene  # noqa: E402

params, cam, gt = make_scene(1_000_000, 1920, 1080, seed=0)
g = ts.GaussianSet(**params)
c = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 1920, 1080, cam["R"], cam["t"])
st = ts.TrainStep(g, ts.TrainConfig(max_iters=30000), extent=4.0)
gt = torch.from_numpy(np.asarray(gt, np.float32)).cuda()
for _ in range(6):
    st.step(c, gt)
torch.cuda.synchronize()
reg = st.regions
nr = 8 if reg.height == 4 else 4
gl = 8 if reg.height == 4 else 16
per_unit = nr // 2
off = st.index.offsets.cpu().numpy()
seg = reg.seg.cpu().numpy()
raise SystemExit("obsolete: K3 files the units longest first (buckets); see tools/unit_probe.py")
span = {}
for t in range(len(off) - 1):
    lo, n = int(off[t]), int(off[t + 1] - off[t])
    if n == 0:
        continue
    prev = np.zeros(nr, np.int64)
    for s in range(1, -(-n // 1024) + 1):
        b = nr * ((lo >> 10) + t + s - 1)
        cur = seg[b:b + nr].astype(np.int64)
        L = np.sort(cur - prev)[::-1]
        prev = cur
        for u in range(2):
            m = int(L[u * per_unit:(u + 1) * per_unit].max())
            span[(t, s - 1, u)] = m + gl - 1 if m > 0 else 0
sp = np.array([span.get((int(x) >> 16, (int(x) >> 1) & 0x7fff, int(x) & 1), 0) for x in units])
order = np.argsort(-sp, kind="stable")
out = torch.zeros_like(st.grad2d)
merges = torch.zeros(1, dtype=torch.int64, device="cuda")


def run(reps=5):
    ts_ = []
    for _ in range(reps):
        reg.ctl[1].zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        backward_regions_raw(st.scratch.rec,
                             st.index.values, st.index.offsets, 1920, 1080, st.targets,
                             st.index.ckpt_base, reg, st.grad_color, None, None, out, merges)
        e1.record()
        torch.cuda.synchronize()
        ts_.append(e0.elapsed_time(e1) * 1e3)
    return np.median(ts_)


orig = reg.units[:n_units].clone()
t_q = run()
reg.units[:n_units] = orig[torch.from_numpy(order).cuda()]
t_l = run()
reg.units[:n_units] = orig
t_q2 = run()
print(f"K4r queue order {t_q:.1f} us, LPT {t_l:.1f} us, queue again {t_q2:.1f} us "
      f"({n_units} units)")
