import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2601_19489_b200 as ts
from paper_2601_19489_b200.synthetic import make_scene
params, cam, gt = make_scene(1_000_000, 1920, 1080, seed=0)
g = ts.GaussianSet(**params)
c = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 1920, 1080, cam["R"], cam["t"])
st = ts.TrainStep(g, ts.TrainConfig(max_iters=30000), extent=4.0)
gt = torch.from_numpy(np.asarray(gt, np.float32)).cuda()
for k in range(300):
    if k % 25 == 0:
        torch.cuda.synchronize(); t0 = time.perf_counter()
    st.step(c, gt)
    if k % 25 == 24:
        torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 25
        b, t, bufs = st.last_view()
        print(k, f"{dt*1e3:.3f} ms", "P", t.n_pairs, "evals", int(bufs.n_considered.sum()), "scale", float(g.log_scales.mean()), "op", float(torch.sigmoid(g.opacity_logits).mean()), "loss", float(st.last_losses[0]))
