"""Where does the e2e (host-fed) step lose time against the device-resident
loop?  Variants over the same TrainStep: resident GT, double-buffered H2D on
a copy stream (bench.py's e2e), serial H2D on the compute stream."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2601_19489_b200 as ts  # noqa: E402
from paper_2601_19489_b200.synthetic import make_scene  # noqa: E402

params, cam, gt = make_scene(1_000_000, 1920, 1080, seed=0)
g = ts.GaussianSet(**params)
c = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 1920, 1080, cam["R"], cam["t"])
st = ts.TrainStep(g, ts.TrainConfig(max_iters=30000), extent=4.0)
gt_host = torch.from_numpy(np.asarray(gt, np.float32)).pin_memory()
gt_dev = gt_host.cuda()
K = 20
for _ in range(5):
    st.step(c, gt_dev)
torch.cuda.synchronize()


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / K * 1e3


def resident():
    for _ in range(K):
        st.step(c, gt_dev)


bufs = [torch.empty_like(gt_dev) for _ in range(2)]


def serial():
    for k in range(K):
        bufs[0].copy_(gt_host, non_blocking=True)
        st.step(c, bufs[0])


cs = torch.cuda.Stream()
copied = [torch.cuda.Event() for _ in range(2)]
consumed = [torch.cuda.Event() for _ in range(2)]


def double():
    with torch.cuda.stream(cs):
        bufs[0].copy_(gt_host, non_blocking=True)
        copied[0].record(cs)
    for k in range(K):
        cur, nxt = k % 2, (k + 1) % 2
        torch.cuda.current_stream().wait_event(copied[cur])
        if k + 1 < K:
            if k >= 1:
                cs.wait_event(consumed[nxt])
            with torch.cuda.stream(cs):
                bufs[nxt].copy_(gt_host, non_blocking=True)
                copied[nxt].record(cs)
        st.step(c, bufs[cur])
        consumed[cur].record()


for name, fn in (("resident", resident), ("double-buffered H2D", double), ("serial H2D", serial),
                 ("resident again", resident)):
    print(f"{name:22s} {timed(fn):.3f} ms/step")
