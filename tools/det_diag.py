"""Find read-before-write / nondeterminism in the deterministic training
step: run it twice sequentially (the second run on recycled, NaN-poisoned
allocator memory) and compare every intermediate buffer after each step."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2601_19489_b200 as ts  # noqa: E402
from oracle.raster import make_scene  # noqa: E402

params, cam, gt = make_scene(20_000, 320, 240, seed=9)
camera = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 320, 240, cam["R"], cam["t"])
g_dev = torch.as_tensor(np.asarray(gt, np.float32), device="cuda")


def run(poison):
    if poison:  # recycle allocator blocks full of NaN
        junk = [torch.full((1 << 26,), float("nan"), device="cuda") for _ in range(8)]
        del junk
    g = ts.GaussianSet(**params)
    st = ts.TrainStep(g, ts.TrainConfig(max_iters=100), deterministic=True)
    snaps = []
    for _ in range(6):
        st.step(camera, g_dev)
        torch.cuda.synchronize()
        o = st.targets
        p = int(st.scratch.totals[1])
        m = int(st.scratch.totals[0])
        snaps.append(dict(color=o.color.clone(), ncons=o.n_considered.clone(),
                          gcol=st.grad_color.clone(), grad2d=st.grad2d[:m].clone(),
                          keys=st.index.keys[:p].clone(), vals=st.index.values[:p].clone(),
                          pos=st.gset.positions.clone(), rec=st.scratch.rec[:m].clone(),
                          ls=st.gset.log_scales.clone(), op=st.gset.opacity_logits.clone()))
    return snaps


A = run(False)
B = run(True)
for step, (a, b) in enumerate(zip(A, B)):
    for k in a:
        x, y = a[k], b[k]
        if x.shape != y.shape:
            print(step, k, "shape", tuple(x.shape), tuple(y.shape))
            continue
        same = torch.equal(x, y)
        print(step, k, "same" if same else
              f"DIFF max {float((x.double() - y.double()).abs().nan_to_num(1e30).max()):.3g} "
              f"n {int((x != y).sum())}")
