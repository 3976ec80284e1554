"""Lockstep efficiency of the region-culled K4's former (tile, segment, half
of the regions) units at C2 after a few training steps: the groups of a
warp run max(L) + kGL - 1 steps; efficiency = sum(L) / (groups x steps).
(K4r now takes length-sorted (tile, segment, region) streams per group:
DESIGN.md §8.)"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_19489_b200 as ts  # noqa: E402
from paper_2601_19489_b200.synthetic import make_scene  # noqa: E402

params, cam, gt = make_scene(1_000_000, 1920, 1080, seed=0)
g = ts.GaussianSet(**params)
c = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 1920, 1080, cam["R"], cam["t"])
st = ts.TrainStep(g, ts.TrainConfig(max_iters=30000), extent=4.0)
gt = torch.from_numpy(np.asarray(gt, np.float32)).cuda()
for _ in range(6):
    st.step(c, gt)
torch.cuda.synchronize()
nr = 8 if st.regions.height == 4 else 4   # regions per tile
gl = 8 if st.regions.height == 4 else 16  # lanes per region pipeline
per_unit = nr // 2
off = st.index.offsets.cpu().numpy()
seg = st.regions.seg.cpu().numpy()
work = steps = 0
lmax_all, eff_units = [], []
for t in range(len(off) - 1):
    lo, n = int(off[t]), int(off[t + 1] - off[t])
    if n == 0:
        continue
    nseg = -(-n // 1024)
    prev = np.zeros(nr, np.int64)
    for s in range(1, nseg + 1):
        b = nr * ((lo >> 10) + t + s - 1)
        cur = seg[b:b + nr].astype(np.int64)
        L = np.sort(cur - prev)[::-1]
        prev = cur
        for u in range(2):
            Lu = L[u * per_unit:(u + 1) * per_unit]
            if Lu.max() == 0:
                continue
            work += int(Lu.sum())
            steps += per_unit * int(Lu.max() + gl - 1)
            lmax_all.append(int(Lu.max()))
print(f"regions/tile {nr}, lanes {gl}: units {len(lmax_all)}, entries {work}, "
      f"group-steps {steps}, lockstep efficiency {work / max(steps, 1):.3f}")
la = np.array(lmax_all)
print("unit max length percentiles:", {q: float(np.percentile(la, q)) for q in (10, 50, 90)})

