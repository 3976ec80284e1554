"""Pins the CPU oracle to the unmodified reference: every oracle function
against the golden vectors made by tests/golden/make_golden.py (CPU only)."""

import numpy as np
import pytest

from conftest import batch_from, golden, rel_err
from oracle import raster as O

BIN_CASES = ("rand", "aniso", "small", "edge")
RASTER_CASES = ("r60", "r128", "deep", "opaque")


@pytest.fixture(scope="module")
def gbin():
    return golden("binning")


@pytest.fixture(scope="module")
def graster():
    return golden("raster")


@pytest.fixture(scope="module")
def gscene():
    return golden("scene")


@pytest.mark.parametrize("case", BIN_CASES)
def test_binning_bit_exact(gbin, case):
    b = batch_from(gbin, case + "_")
    x_min, _, _, y_max, rect = O.snugboxes(b)
    assert np.array_equal(rect, gbin[case + "_rect"])
    assert np.array_equal(x_min, gbin[case + "_xmin"])
    assert np.array_equal(y_max, gbin[case + "_ymax"])
    for idx in (O.bin_sequential(b), O.bin_load_balanced(b)):
        assert np.array_equal(idx["keys"], gbin[case + "_seq_keys"])
        assert np.array_equal(idx["values"], gbin[case + "_seq_values"])
        assert np.array_equal(idx["offsets"], gbin[case + "_seq_offsets"])
        assert O.checksum(idx) == str(gbin[case + "_seq_checksum"])


def test_edge_cases_pinned(gbin):
    # tangency inclusive (test_binning.py:152-164), off-screen emits nothing
    vals = gbin["edge_seq_values"]
    keys = gbin["edge_seq_keys"]
    tiles_of = lambda r: set(int(k >> np.uint64(32)) for k, v in zip(keys, vals) if v == r)
    assert 1 * 8 + 2 in tiles_of(0)          # tile (2, 1) at t = 4
    assert 2 * 8 + 2 in tiles_of(1)          # corner tile (2, 2) at t = 8
    assert tiles_of(3) == set()              # off-screen
    assert tiles_of(2) == {2 * 8 + 2}        # t = 0: centre tile only


def _raster_inputs(g, name):
    b = batch_from(g, name + "_")
    idx = dict(keys=g[name + "_keys"], values=g[name + "_values"],
               offsets=g[name + "_offsets"], tiles_x=-(-b["width"] // 16),
               tiles_y=-(-b["height"] // 16))
    return b, idx, g[name + "_colors"], g[name + "_bg"]


@pytest.mark.parametrize("case", RASTER_CASES)
def test_render_and_backward_match_reference(graster, case):
    g = graster
    b, idx, colors, bg = _raster_inputs(g, case)
    ob = O.bin_sequential(b)
    assert np.array_equal(ob["keys"], idx["keys"])
    bufs = O.render(b, idx, colors, bg)
    for k in ("color", "depth", "final_T"):
        assert np.abs(bufs[k] - g[f"{case}_{k}"]).max() < 1e-12, k
    for k in ("n_contrib", "n_considered"):
        assert np.array_equal(bufs[k], g[f"{case}_{k}"]), k
    for t, ck in bufs["checkpoints"].items():
        ref = g[f"{case}_ckpt_{t}"]
        assert np.abs(ck.reshape(ref.shape) - ref).max() < 1e-12
    out = O.backward_per_gaussian(bufs, b, idx, colors, g[case + "_gc"], g[case + "_gd"],
                                  g[case + "_gt"])
    for k in ("d_means2d", "d_conics", "d_opacities", "d_colors", "d_depths"):
        assert rel_err(out[k], g[f"{case}_pg_{k}"]) < 1e-10, k
        # and transitively the reference's per-pixel path (criterion 4)
        assert rel_err(out[k], g[f"{case}_pp_{k}"]) < 1e-5, k
    assert out["merges"] == int(g[case + "_merges"])


@pytest.mark.parametrize("case", ("s0", "s1", "sh"))
def test_scene_end_to_end(gscene, case):
    g = gscene
    params = {k: g[f"{case}_p_{k}"] for k in ("positions", "log_scales", "rotations",
                                             "opacity_logits", "colors")}
    f = g[f"{case}_cam_f"]
    cam = dict(fx=f[0], fy=f[1], cx=f[2], cy=f[3], width=int(f[4]), height=int(f[5]),
               R=g[f"{case}_cam_R"], t=g[f"{case}_cam_t"])
    batch, colors = O.project(params, cam, 0.01)
    ref_b = batch_from(g, case + "_b_")
    for k in ("means2d", "conics", "level_t", "depths", "opacities"):
        assert rel_err(batch[k], ref_b[k]) < 1e-12, k
    assert np.array_equal(batch["source_ids"], ref_b["source_ids"])
    assert rel_err(colors, g[f"{case}_colors"]) < 1e-12
    # raster on the FP32-rounded batch, as the golden did
    b32 = {k: (np.asarray(v, np.float32).astype(np.float64) if isinstance(v, np.ndarray)
               and v.dtype == np.float64 else v) for k, v in batch.items()}
    c32 = np.asarray(colors, np.float32).astype(np.float64)
    idx = O.bin_sequential(b32)
    assert np.array_equal(idx["keys"], g[f"{case}_keys"])
    assert np.array_equal(idx["values"], g[f"{case}_values"])
    bufs = O.render(b32, idx, c32, np.zeros(3))
    for k in ("color", "depth", "final_T"):
        assert np.abs(bufs[k] - g[f"{case}_{k}"]).max() < 1e-12, k
    e, l1, ssim, gcol = O.photometric(bufs["color"], g[f"{case}_gt"])
    assert np.allclose([e, l1, ssim], g[f"{case}_loss"], rtol=1e-12)
    assert rel_err(gcol, g[f"{case}_gcol"]) < 1e-10
    g2 = O.backward_per_gaussian(bufs, b32, idx, c32, gcol)
    for k in ("d_means2d", "d_conics", "d_opacities", "d_colors", "d_depths"):
        assert rel_err(g2[k], g[f"{case}_g2_{k}"]) < 1e-10, k
    if case != "sh":
        g3 = O.project_vjp(params, cam, batch, g2)
        for k in ("positions", "log_scales", "rotations", "opacity_logits"):
            assert rel_err(g3[k], g[f"{case}_g3_{k}"]) < 1e-9, k


def test_projection_vjp_and_pose():
    g = golden("projection")
    params = {k[2:]: v for k, v in g.items() if k.startswith("p_")}
    f = g["cam_f"]
    cam = dict(fx=f[0], fy=f[1], cx=f[2], cy=f[3], width=64, height=64, R=g["cam_R"],
               t=g["cam_t"])
    batch, _ = O.project(params, cam, 0.1)
    ref_b = batch_from(g, "b_")
    assert np.array_equal(batch["source_ids"], ref_b["source_ids"])
    assert 3 not in batch["source_ids"] and 5 not in batch["source_ids"]
    g2 = dict(d_means2d=g["g_means"], d_conics=g["g_conics"], d_depths=g["g_depths"],
              d_opacities=g["g_opac"], d_colors=np.zeros((len(g["g_depths"]), 3)))
    g3 = O.project_vjp(params, cam, batch, g2, near=0.1)
    for k in ("positions", "log_scales", "rotations", "opacity_logits"):
        assert rel_err(g3[k], g[f"g3_{k}"]) < 1e-10, k
    rot, trans = O.pose_from_sums(g3["pose_S1"], g3["pose_S2"], cam["R"])
    assert rel_err(np.concatenate([rot, trans]), g["pose"]) < 1e-10


def test_adam_sequence():
    g = golden("adam")
    names = ("positions", "rotations", "colors")
    lrs = {"positions": 1e-2, "rotations": 0.1, "colors": 3e-3}
    p = {k: g[f"init_{k}"].copy() for k in names}
    m = {k: np.zeros_like(v) for k, v in p.items()}
    v = {k: np.zeros_like(x) for k, x in p.items()}
    for step in range(4):
        skipped = 0
        for k in names:
            skipped += O.adam_step(p[k], g[f"g{step}_{k}"], m[k], v[k], step + 1, lrs[k],
                                   renormalize=(k == "rotations"))
        assert skipped == int(g[f"skipped{step}"])
        for k in names:
            assert np.array_equal(p[k], g[f"p{step}_{k}"]), (step, k)
            assert np.array_equal(m[k], g[f"m{step}_{k}"])


def test_photometric_loss():
    g = golden("loss")
    e, l1, ssim, grad = O.photometric(g["rendered"], g["gt"], 0.2)
    assert np.allclose([e, l1, ssim], g["values"], rtol=1e-13)
    assert rel_err(grad, g["grad"]) < 1e-12
