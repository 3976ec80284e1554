"""End-to-end parity on canonical synthetic scenes:
the whole device path -- K1 projection, K2 binning, K3 render, loss, K4
backward, K4b+K5 fused VJP+Adam -- against the oracle on the same inputs, and
against the reference's golden vectors for the small scenes."""

import numpy as np
import pytest
import torch

from conftest import batch_from, golden, host_batch, host_index, np64, rel_err
from oracle import raster as O

pytestmark = pytest.mark.gpu

RENDER_ATOL = 2e-5
GRAD_RTOL = 1e-4
VJP_RTOL = 5e-4


def _setup(n, w, h, seed=0, clustered=False, sh_degree=0):
    import paper_2601_19489_b200 as ts
    params, cam, gt = O.make_scene(n, w, h, seed=seed, clustered=clustered,
                                   sh_degree=sh_degree)
    gset = ts.GaussianSet(**params)
    camera = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], w, h, cam["R"], cam["t"])
    return ts, params, cam, gt, gset, camera


@pytest.mark.parametrize("case", ("s0", "s1", "sh"))
def test_golden_scene(case):
    import paper_2601_19489_b200 as ts
    g = golden("scene")
    params = {k: g[f"{case}_p_{k}"] for k in ("positions", "log_scales", "rotations",
                                             "opacity_logits", "colors")}
    f = g[f"{case}_cam_f"]
    gset = ts.GaussianSet(**params)
    camera = ts.Camera(float(f[0]), float(f[1]), float(f[2]), float(f[3]), int(f[4]), int(f[5]),
                       g[f"{case}_cam_R"], g[f"{case}_cam_t"])
    batch = ts.project(gset, camera)
    ref = batch_from(g, case + "_b_")
    assert np.array_equal(np64(batch.source_ids), ref["source_ids"])
    for k in ("means2d", "conics", "level_t", "depths", "opacities"):
        assert rel_err(np64(getattr(batch, k)), ref[k]) < 2e-5, k
    assert rel_err(np64(batch.colors), g[f"{case}_colors"]) < 2e-5


def test_c1_forward_backward_vs_oracle():
    """Config 1: 10k Gaussians, 256x256, one forward + backward."""
    ts, params, cam, gt, gset, camera = _setup(10_000, 256, 256)
    cfg = ts.TrainConfig()
    vr = ts.render_view(gset, camera, cfg)
    hb = host_batch(vr.batch)
    hi = host_index(vr.tiles)
    ref_idx = O.bin_sequential(hb)
    assert np.array_equal(hi["keys"], ref_idx["keys"])
    assert np.array_equal(hi["values"], ref_idx["values"])
    assert np.array_equal(hi["offsets"], ref_idx["offsets"])
    colors = np64(vr.colors)
    ob = O.render(hb, ref_idx, colors, np.zeros(3))
    assert np.abs(np64(vr.buffers.color) - ob["color"]).max() < RENDER_ATOL
    assert np.abs(np64(vr.buffers.final_T) - ob["final_T"]).max() < RENDER_ATOL
    flips = int((np64(vr.buffers.n_considered) != ob["n_considered"]).sum())
    assert flips == 0, f"{flips} threshold flips"
    camera.gt_image = gt
    report, g2 = ts.view_loss_and_grads(camera, cfg, vr, 0.0)
    e, l1, ssim, gcol = O.photometric(ob["color"], gt)
    assert abs(report.photometric - e) < 1e-5 and abs(report.ssim - ssim) < 1e-5
    og = O.backward_per_gaussian(ob, hb, ref_idx, colors, gcol)
    for k in ("d_means2d", "d_conics", "d_opacities", "d_colors"):
        err = rel_err(np64(getattr(g2, k)), og[k])
        assert err < GRAD_RTOL, (k, err)
    assert g2.merges == og["merges"]
    grads = ts._full_grads(gset, camera, cfg, None, vr, g2)
    o3 = O.project_vjp(params, cam, hb, og)
    for k in ("positions", "log_scales", "rotations", "opacity_logits", "colors"):
        assert rel_err(np64(grads[k]), o3[k]) < VJP_RTOL, k


def test_fused_train_step_matches_separate_path(monkeypatch):
    """K4b+K5 fused == project_vjp then Adam.step (same device gradients).
    Both paths run the per-tile K4 (the public backward_per_gaussian's), so
    the Grad2D they feed are the same sums; the region-culled K4 of the
    default training step has its own parity tests (test_gpu_regions.py)."""
    from paper_2601_19489_b200 import backward as bw
    monkeypatch.setattr(bw, "K4_FORM", "tiles")
    ts, params, cam, gt, gset, camera = _setup(20_000, 320, 200, seed=2)
    cfg = ts.TrainConfig(max_iters=100)
    gset_b = gset.copy()
    gt_t = torch.tensor(gt, dtype=torch.float32, device="cuda")
    step = ts.TrainStep(gset, cfg, extent=4.0)
    loss = step.step(camera, gt_t)
    assert torch.isfinite(loss)
    # separate path on the copy
    camera.gt_image = gt
    vr = ts.render_view(gset_b, camera, cfg)
    _, g2 = ts.view_loss_and_grads(camera, cfg, vr, 0.0)
    grads = ts._full_grads(gset_b, camera, cfg, None, vr, g2)
    opt = ts.Adam()
    lr = {"positions": ts.position_lr(1.6e-4 * 4.0, 1, cfg.max_iters)}
    opt.step(gset_b.params(), {k: grads[k] for k in gset_b.params()}, lr)
    for k in gset.params():
        assert rel_err(np64(gset.params()[k]), np64(gset_b.params()[k])) < 1e-5, k


def test_c2_scale_binning_exact_and_render_sample():
    """Config 2 size (1M Gaussians, 1080p): keys/values/offsets bit-exact vs the
    oracle on the full batch; render on a sample of tiles vs the oracle."""
    ts, params, cam, gt, gset, camera = _setup(1_000_000, 1920, 1080)
    cfg = ts.TrainConfig()
    vr = ts.render_view(gset, camera, cfg)
    hb = host_batch(vr.batch)
    ref_idx = O.bin_sequential(hb)
    hi = host_index(vr.tiles)
    assert hi["keys"].shape == ref_idx["keys"].shape
    assert O.checksum(hi) == O.checksum(ref_idx)
    assert vr.tiles.checksum() == O.checksum(ref_idx)
    # sortedness / range properties at full size
    tiles = hi["keys"] >> np.uint64(32)
    assert np.all(np.diff(tiles.astype(np.int64)) >= 0)
    assert hi["offsets"][-1] == len(hi["keys"])
    # sampled-tile render parity: oracle restricted to 40 tiles
    rng = np.random.default_rng(0)
    busy = np.flatnonzero(np.diff(ref_idx["offsets"]) > 0)
    pick = rng.choice(busy, 40, replace=False)
    sub = dict(ref_idx)
    offs = np.zeros_like(ref_idx["offsets"])
    keep_rows = []
    # build an index holding only the sampled tiles
    cur = 0
    order = []
    for t in range(len(offs) - 1):
        offs[t] = cur
        if t in set(pick.tolist()):
            lo, hi_ = ref_idx["offsets"][t], ref_idx["offsets"][t + 1]
            order.append(np.arange(lo, hi_))
            cur += hi_ - lo
    offs[-1] = cur
    order = np.concatenate(order)
    sub.update(keys=ref_idx["keys"][order], values=ref_idx["values"][order], offsets=offs)
    ob = O.render(hb, sub, np64(vr.colors), np.zeros(3))
    for t in pick:
        ty, tx = divmod(int(t), sub["tiles_x"])
        sl = (slice(ty * 16, ty * 16 + 16), slice(tx * 16, tx * 16 + 16))
        assert np.abs(np64(vr.buffers.color[sl]) - ob["color"][sl]).max() < 5e-5
        assert np.abs(np64(vr.buffers.n_considered[sl]) - ob["n_considered"][sl]).max() <= 1
    del keep_rows


def test_c3_clustered_heavy_tiles_binning_exact_and_bounded_work():
    """Config 3 (3M Gaussians, half clustered in depth): heavy tiles (>100k
    entries).  Keys/values/offsets bit-exact vs the oracle; render and
    backward complete with finite outputs and per-tile work bounded by
    termination (max n_considered << max tile length)."""
    ts, params, cam, gt, gset, camera = _setup(3_000_000, 1920, 1080, seed=0, clustered=True)
    cfg = ts.TrainConfig()
    vr = ts.render_view(gset, camera, cfg)
    hb = host_batch(vr.batch)
    ref_idx = O.bin_sequential(hb)
    assert vr.tiles.checksum() == O.checksum(ref_idx)
    counts = np.diff(ref_idx["offsets"])
    assert counts.max() > 100_000
    ncons = np64(vr.buffers.n_considered)
    assert ncons.max() < counts.max() // 10
    camera.gt_image = gt
    report, g2 = ts.view_loss_and_grads(camera, cfg, vr, 0.0)
    assert np.isfinite(report.total)
    assert np.isfinite(np64(g2.packed)).all()
    assert g2.merges == vr.tiles.n_pairs


@pytest.mark.parametrize("k4", ["auto", "regions"])
def test_graph_replayed_train_step_matches_eager(k4, monkeypatch):
    """TrainStep(graphs=True) replays one captured CUDA graph per (camera, GT)
    with the per-step Adam scalars and depth weight fed through pinned-memory
    copy nodes; parameters after several steps (alternating two GT buffers,
    depth supervision on) match the eager step within FP32 tolerance.
    k4="regions" forces the region-culled K3/K4r pair on this small frame
    (the training step's form at C2 size), incl. its depth channel."""
    import torch
    import paper_2601_19489_b200 as ts
    if k4 == "regions":
        from paper_2601_19489_b200 import backward as bw
        monkeypatch.setattr(bw, "REGIONS_MIN_PAIRS", 0)
    from oracle.raster import make_scene
    params, cam, gt = make_scene(20_000, 320, 240, seed=8)
    camera = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 320, 240, cam["R"], cam["t"])
    gts = [torch.as_tensor(np.asarray(gt, np.float32), device="cuda")] * 2
    gts[1] = gts[0].flip(1).contiguous()
    prior = torch.full((240, 320), 4.0, device="cuda")
    valid = torch.ones((240, 320), dtype=torch.bool, device="cuda")
    out = {}
    losses = {}
    for run, graphs in (("eager", False), ("eager2", False), ("graph", True)):
        g = ts.GaussianSet(**params)
        st = ts.TrainStep(g, ts.TrainConfig(max_iters=100), graphs=graphs)
        ls = []
        for k in range(6):
            e = st.step(camera, gts[k % 2], depth_weight=0.05 * (k % 3), depth_prior=prior,
                        depth_valid=valid)
            ls.append(float(e))
        torch.cuda.synchronize()
        out[run] = g.to_numpy()
        losses[run] = ls
        assert (st.regions is not None) == (k4 == "regions")
        if graphs:
            assert len(st._graph_cache) >= 2  # two GT buffers (and depth on/off)
    assert np.allclose(losses["eager"], losses["graph"], rtol=1e-5, atol=1e-7)
    # K4 merges with float atomics, so two eager runs already differ in the
    # last ulps and Adam's first steps (a move of ~lr * sign(g) per row)
    # amplify that where g ~ 0: the graph run must differ from the eager run
    # no more than a second eager run does
    lrs = {"positions": 1.6e-4 * 4.0, "log_scales": 5e-3, "rotations": 1e-3,
           "opacity_logits": 5e-2, "colors": 2.5e-3}
    for k in out["eager"]:
        a = out["eager"][k]
        tol = 1e-5 * max(np.abs(a).max(), 1.0)
        dg = np.abs(a - out["graph"][k]).reshape(len(a), -1).max(axis=1)
        de = np.abs(a - out["eager2"][k]).reshape(len(a), -1).max(axis=1)
        assert dg.max() <= 12 * lrs[k], k
        assert (dg > tol).mean() <= 2.0 * (de > tol).mean() + 0.005, k


def test_deterministic_train_step_is_bitwise_reproducible():
    """TrainStep(deterministic=True): two runs from the same state give
    bitwise-identical parameters (the reference's determinism contract,
    test_trainer.py:74-82), eager and graph-replayed alike."""
    import torch
    import paper_2601_19489_b200 as ts
    from oracle.raster import make_scene
    params, cam, gt = make_scene(20_000, 320, 240, seed=9)
    camera = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 320, 240, cam["R"], cam["t"])
    g_dev = torch.as_tensor(np.asarray(gt, np.float32), device="cuda")
    runs = []
    for graphs in (False, False, True):
        g = ts.GaussianSet(**params)
        st = ts.TrainStep(g, ts.TrainConfig(max_iters=100), deterministic=True, graphs=graphs)
        for _ in range(5):
            st.step(camera, g_dev)
        torch.cuda.synchronize()
        runs.append(g.to_numpy())
    for k in runs[0]:
        assert np.array_equal(runs[0][k], runs[1][k]), k
        assert np.array_equal(runs[0][k], runs[2][k]), k


@pytest.mark.parametrize("graphs", [False, True])
def test_gt_refilled_after_gt_consumed_trains_like_resident_gt(graphs):
    """A host-fed loop that refills each of two GT buffers as soon as
    TrainStep.gt_consumed fires (the copy of view k + 2 overlaps step k's
    backward; bench.py's e2e loop) trains exactly like device-resident GT
    images: deterministic merge, a different GT every step, bitwise-equal
    parameters and losses.  A GT buffer overwritten before its step's loss
    kernels read it would change them."""
    import torch
    import paper_2601_19489_b200 as ts
    from oracle.raster import make_scene
    params, cam, gt = make_scene(20_000, 320, 240, seed=11)
    camera = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 320, 240, cam["R"], cam["t"])
    rng = np.random.default_rng(5)
    host = [torch.from_numpy(np.clip(np.asarray(gt, np.float32)
                                     + rng.normal(0, 0.1, gt.shape).astype(np.float32), 0, 1))
            .pin_memory() for _ in range(5)]
    steps = 8
    # resident: every step's GT already on the device
    g = ts.GaussianSet(**params)
    st = ts.TrainStep(g, ts.TrainConfig(max_iters=100), deterministic=True, graphs=graphs)
    dev = [h.cuda() for h in host]
    ref_losses = [float(st.step(camera, dev[k % 5])) for k in range(steps)]
    torch.cuda.synchronize()
    ref = g.to_numpy()
    # host-fed: two device buffers refilled after gt_consumed
    g = ts.GaussianSet(**params)
    st = ts.TrainStep(g, ts.TrainConfig(max_iters=100), deterministic=True, graphs=graphs)
    cs = torch.cuda.Stream()
    bufs = [torch.empty_like(dev[0]) for _ in range(2)]
    copied = [torch.cuda.Event() for _ in range(2)]
    with torch.cuda.stream(cs):
        for b in range(2):
            bufs[b].copy_(host[b], non_blocking=True)
            copied[b].record(cs)
    losses = []
    for k in range(steps):
        cur = k % 2
        torch.cuda.current_stream().wait_event(copied[cur])
        losses.append(st.step(camera, bufs[cur]).clone())  # a replay reuses its output
        if k + 2 < steps:
            cs.wait_event(st.gt_consumed)
            with torch.cuda.stream(cs):
                bufs[cur].copy_(host[(k + 2) % 5], non_blocking=True)
                copied[cur].record(cs)
    torch.cuda.synchronize()
    assert [float(e) for e in losses] == ref_losses
    out = g.to_numpy()
    for name in ref:
        assert np.array_equal(out[name], ref[name]), name
