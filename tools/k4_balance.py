"""K4 schedule model at C2: per (tile, supergroup) unit cost = active pixels
+ 31 fill steps (systolic steps); efficiency of 4 warps per tile CTA (greedy,
dynamic grab) vs a global warp queue.  usage: python tools/k4_balance.py [c2|c3]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_19489_b200 as ts  # noqa: E402
from paper_2601_19489_b200.synthetic import make_scene  # noqa: E402

cfg = {"c2": (1_000_000, False), "c3": (3_000_000, True)}[sys.argv[1] if len(sys.argv) > 1 else "c2"]
params, cam, gt = make_scene(cfg[0], 1920, 1080, seed=0, clustered=cfg[1])
g = ts.GaussianSet(**params)
c = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 1920, 1080, cam["R"], cam["t"])
st = ts.TrainStep(g, ts.TrainConfig(max_iters=30000), extent=4.0)
gt_t = torch.from_numpy(np.asarray(gt, np.float32)).cuda()
for _ in range(6):
    st.step(c, gt_t)
b, tiles, bufs = st.last_view()
nc = bufs.n_considered.cpu().numpy()
H, W = nc.shape
ty, tx = (H + 15) // 16, (W + 15) // 16
pad = np.zeros((ty * 16, tx * 16), np.int64)
pad[:H, :W] = nc
t = pad.reshape(ty, 16, tx, 16).transpose(0, 2, 1, 3).reshape(ty * tx, 256)
mx = t.max(1)
nsup = (mx + 63) // 64
costs, mk, tot = [], 0.0, 0.0
for i in range(len(t)):
    u = [int((t[i] > 64 * G).sum()) + 31 for G in range(nsup[i])]
    if not u:
        continue
    costs += u
    w = [0] * 4
    for x in u:  # dynamic grab: next unit to the least-loaded warp
        w[w.index(min(w))] += x
    mk += max(w)
    tot += sum(u)
steps = sum(costs)
print(f"units {len(costs)}  steps {steps}  mean n_act+31 {np.mean(costs):.1f}")
print(f"per-tile CTA (4 warps): warp-slot efficiency {tot / (4 * mk):.3f}")
print(f"fill share {31 * len(costs) / steps:.3f}")
