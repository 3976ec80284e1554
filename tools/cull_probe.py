import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2601_19489_b200 as ts
from paper_2601_19489_b200 import _lib
from paper_2601_19489_b200.synthetic import make_scene
params, cam, gt = make_scene(1_000_000, 1920, 1080, seed=0)
g = ts.GaussianSet(**params)
c = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 1920, 1080, cam["R"], cam["t"])
st = ts.TrainStep(g, ts.TrainConfig(max_iters=30000), extent=4.0)
gt = torch.from_numpy(np.asarray(gt, np.float32)).cuda()
st.step(c, gt); torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * 2)()
lib.tsr_cull_stats_read(buf)
print("chunks positions considered by warps:", buf[0], "hits:", buf[1], "frac", buf[1] / buf[0])
b, t, bufs = st.last_view()
print("sum n_considered", int(bufs.n_considered.sum()), "sum n_contrib", int(bufs.n_contrib.sum()))
