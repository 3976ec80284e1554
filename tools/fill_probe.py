"""K4 systolic step accounting at C2: steps per supergroup with the 32-lane
pipeline (n_act + 31) vs two 16-lane pipelines per supergroup (n_act + 15),
from the per-pixel n_considered of a training step."""
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
b, t, bufs = st.last_view()
nc = bufs.n_considered.cpu().numpy().reshape(1080, 1920)
H, W = 1088, 1920
pad = np.zeros((H, W), np.int64)
pad[:1080] = nc
tiles = pad.reshape(68, 16, 120, 16).transpose(0, 2, 1, 3).reshape(-1, 256)
mx = tiles.max(1)
cur = new = acts = 0
for G in range(int(np.ceil(mx.max() / 64))):
    act = (tiles > 64 * G).sum(1)
    live = act[mx > 64 * G]
    acts += live.sum()
    cur += (((live + 31 + 3) // 4) * 4).sum()
    new += (((live + 15 + 3) // 4) * 4).sum()
print("sum n_act", acts, "steps 32-lane", cur, "steps 16-lane", new, "saving", 1 - new / cur)
print("evals", int(nc.sum()))
