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
st = ts.TrainStep(g, ts.TrainConfig(max_iters=30000), extent=4.0, graphs=True)
gt_host = torch.from_numpy(np.asarray(gt, np.float32)).pin_memory()
gt_dev = gt_host.cuda()
K = 20
for _ in range(5):
    st.step(c, gt_dev)
torch.cuda.synchronize()


# every variant replays the same training segment (the scene trains during
# the run and per-step work drifts: tools/drift_probe.py)
snap = {k: v.clone() for k, v in g.params().items()}
snap_m = {k: v.clone() for k, v in st.opt._m.items()}
snap_v = {k: v.clone() for k, v in st.opt._v.items()}
snap_steps = dict(st.opt._steps)
snap_it = st.iteration


def restore():
    torch.cuda.synchronize()
    for k, v in g.params().items():
        v.copy_(snap[k])
    for k in snap_m:
        st.opt._m[k].copy_(snap_m[k])
        st.opt._v[k].copy_(snap_v[k])
    st.opt._steps.update(snap_steps)
    st.iteration = snap_it
    torch.cuda.synchronize()


def timed(fn):
    fn()  # graphs for every buffer captured before timing
    restore()
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


loss_host = torch.zeros(K, dtype=torch.float32).pin_memory()


def double_d2h(on_copy_stream):
    """bench.py's e2e loop: double-buffered GT H2D plus a per-step loss D2H,
    on the compute stream (as bench.py) or on the copy stream after the step."""
    done = [torch.cuda.Event() for _ in range(2)]
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
        loss = st.step(c, bufs[cur])
        consumed[cur].record()
        if on_copy_stream:
            cs.wait_event(consumed[cur])
            with torch.cuda.stream(cs):
                loss_host[k:k + 1].copy_(loss.reshape(1), non_blocking=True)
                done[cur].record(cs)
        else:
            loss_host[k:k + 1].copy_(loss.reshape(1), non_blocking=True)


def early_refill():
    """GT buffer refilled once the step's loss kernels have read it
    (TrainStep.gt_consumed): the copy for step k + 2 runs under step k's
    backward."""
    with torch.cuda.stream(cs):
        bufs[0].copy_(gt_host, non_blocking=True)
        copied[0].record(cs)
        bufs[1].copy_(gt_host, non_blocking=True)
        copied[1].record(cs)
    for k in range(K):
        cur = k % 2
        torch.cuda.current_stream().wait_event(copied[cur])
        loss = st.step(c, bufs[cur])
        if k + 2 < K:
            cs.wait_event(st.gt_consumed)
            with torch.cuda.stream(cs):
                bufs[cur].copy_(gt_host, non_blocking=True)
                copied[cur].record(cs)
        loss_host[k:k + 1].copy_(loss.reshape(1), non_blocking=True)


def replay_only():
    """The cached step graph replayed K times: no per-step scalar upload or
    host bookkeeping (fixed scalars: timing only)."""
    g0 = next(iter(st._graph_cache.values()))[0]
    for _ in range(K):
        g0.replay()


for name, fn in (("resident", resident), ("graph replay only", replay_only),
                 ("double-buffered H2D", double), ("serial H2D", serial),
                 ("early refill (gt_consumed)", early_refill),
                 ("double + D2H (compute)", lambda: double_d2h(False)),
                 ("double + D2H (copy)", lambda: double_d2h(True)),
                 ("resident again", resident)):
    print(f"{name:22s} {timed(fn):.3f} ms/step")
