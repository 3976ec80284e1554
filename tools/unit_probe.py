"""Distribution of the region-culled K4's unit spans (max list length of the
unit's two regions) at C2 after a few training steps."""
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
off = st.index.offsets.cpu().numpy()
seg = st.regions.seg.cpu().numpy()
spans = []
for t in range(len(off) - 1):
    lo, n = int(off[t]), int(off[t + 1] - off[t])
    if n == 0:
        continue
    nseg = -(-n // 1024)
    prev = np.zeros(4, np.int64)
    for s in range(1, nseg + 1):
        cur = seg[4 * ((lo >> 10) + t + s - 1): 4 * ((lo >> 10) + t + s - 1) + 4].astype(np.int64)
        L = np.sort(cur - prev)[::-1]
        prev = cur
        for pair in (L[:2], L[2:]):
            spans.append(int(pair.max()))
spans = np.array(spans)
nz = spans[spans > 0]
print("units", len(spans), "nonempty", len(nz), "sum span", int(nz.sum()), "fill 15/unit", 15 * len(nz))
for q in (5, 10, 25, 50, 75, 90):
    print(f"p{q}", np.percentile(nz, q))
print("units with span < 17:", int((nz < 17).sum()), " < 32:", int((nz < 32).sum()))
pad32 = np.maximum(nz, 32).sum()
print("current steps ~", int((nz + 15).sum()), " chained (pad 32) ~", int(pad32 + 15 * 0))
