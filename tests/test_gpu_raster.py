"""K3/K4 parity: render and per-Gaussian backward vs the reference's golden
vectors (FP32 tolerances stated per assertion) and closed forms
(test_forward.py / test_backward.py counterparts)."""

import numpy as np
import pytest

from conftest import batch_from, dev_batch, golden, host_index, np64, rel_err

pytestmark = pytest.mark.gpu

RASTER_CASES = ("r60", "r128", "deep", "opaque")
# FP32 accumulation over <= a few hundred list entries, ex2.approx alphas
RENDER_ATOL = 2e-5
GRAD_RTOL = 1e-4          # max|x-y| / max|y|, the reference's metric


@pytest.fixture(scope="module")
def graster():
    return golden("raster")


def _run(g, case, with_depth=True, with_T=True):
    import paper_2601_19489_b200 as ts
    b = batch_from(g, case + "_")
    db = dev_batch(b)
    idx = ts.bin_sequential(db)
    h = host_index(idx)
    assert np.array_equal(h["keys"], g[case + "_keys"].astype(np.uint64))
    bufs = ts.render(db, idx, g[case + "_colors"], g[case + "_bg"])
    g2 = ts.backward_per_gaussian(bufs, db, idx, g[case + "_colors"], g[case + "_gc"],
                                  g[case + "_gd"] if with_depth else None,
                                  g[case + "_gt"] if with_T else None)
    return db, idx, bufs, g2


@pytest.mark.parametrize("case", RASTER_CASES)
def test_render_matches_reference(graster, case):
    g = graster
    _, idx, bufs, _ = _run(g, case)
    assert np.abs(np64(bufs.color) - g[case + "_color"]).max() < RENDER_ATOL
    assert np.abs(np64(bufs.final_T) - g[case + "_final_T"]).max() < RENDER_ATOL
    dref = g[case + "_depth"]
    assert np.abs(np64(bufs.depth) - dref).max() < RENDER_ATOL * max(1.0, np.abs(dref).max())
    assert np.array_equal(np64(bufs.n_contrib), g[case + "_n_contrib"])
    assert np.array_equal(np64(bufs.n_considered), g[case + "_n_considered"])
    # checkpoints, on the records each pixel actually reached
    nc = g[case + "_n_considered"]
    for t, ck in bufs.checkpoints_dict(idx).items():
        ref = g[f"{case}_ckpt_{t}"]
        ty, tx = divmod(t, idx.tiles_x)
        ncons = nc[ty * 16: ty * 16 + ref.shape[2], tx * 16: tx * 16 + ref.shape[3]]
        got = np64(ck)
        for r in range(ref.shape[0]):
            reached = ncons >= 32 * (r + 1)
            if reached.any():
                err = np.abs(got[r][:, reached] - ref[r][:, reached]).max()
                assert err < RENDER_ATOL * 10, (t, r, err)


@pytest.mark.parametrize("case", RASTER_CASES)
def test_backward_matches_reference(graster, case):
    g = graster
    _, idx, _, g2 = _run(g, case)
    for k in ("d_means2d", "d_conics", "d_opacities", "d_colors", "d_depths"):
        err = rel_err(np64(getattr(g2, k)), g[f"{case}_pg_{k}"])
        assert err < GRAD_RTOL, (k, err)
        # transitively the reference's per-pixel path (criterion 4)
        assert rel_err(np64(getattr(g2, k)), g[f"{case}_pp_{k}"]) < GRAD_RTOL, k
    assert g2.merges == int(g[case + "_merges"]) == idx.n_pairs


def test_missing_checkpoints_is_hard_error(graster):
    import paper_2601_19489_b200 as ts
    g = graster
    db = dev_batch(batch_from(g, "deep_"))
    idx = ts.bin_sequential(db)
    bufs = ts.render(db, idx, g["deep_colors"], g["deep_bg"], record_checkpoints=False)
    with pytest.raises(ts.CheckpointsMissingError):
        ts.backward_per_gaussian(bufs, db, idx, g["deep_colors"], np.ones((16, 16, 3)))


def test_zero_upstream_gives_zero_grads_and_no_merges(graster):
    import paper_2601_19489_b200 as ts
    g = graster
    db = dev_batch(batch_from(g, "r60_"))
    idx = ts.bin_sequential(db)
    bufs = ts.render(db, idx, g["r60_colors"], g["r60_bg"])
    g2 = ts.backward_per_gaussian(bufs, db, idx, g["r60_colors"], np.zeros((32, 32, 3)))
    assert not np.any(np64(g2.packed)) and g2.merges == 0


def _centered(n, opacities, depths, sigma=6.0, w=32, h=32):
    a = 1.0 / sigma ** 2
    t = [max(0.0, 2 * np.log(255 * o)) for o in opacities]
    return dict(means2d=np.array([[w / 2 + 0.5, h / 2 + 0.5]] * n),
                conics=np.array([[a, 0.0, a]] * n), level_t=np.array(t),
                depths=np.array(depths, float), opacities=np.array(opacities, float),
                source_ids=np.arange(n), width=w, height=h)


def test_closed_forms():
    """test_forward.py:38-56: alpha 0.5 at the centre; two-splat compositing."""
    import paper_2601_19489_b200 as ts
    b = dev_batch(_centered(1, [0.5], [2.0]))
    bufs = ts.render(b, ts.bin_sequential(b), np.ones((1, 3)), np.zeros(3))
    assert abs(float(bufs.color[16, 16, 0]) - 0.5) < 1e-6
    assert abs(float(bufs.final_T[16, 16]) - 0.5) < 1e-6
    assert int(bufs.n_contrib[16, 16]) == 1
    b2 = dev_batch(_centered(2, [0.5, 0.5], [1.5, 3.0]))
    bufs = ts.render(b2, ts.bin_sequential(b2), np.array([[1.0, 0, 0], [0, 1.0, 0]]), np.zeros(3))
    assert np.allclose(np64(bufs.color[16, 16]), [0.5, 0.25, 0.0], atol=1e-6)
    assert abs(float(bufs.depth[16, 16]) - (0.5 * 1.5 + 0.25 * 3.0)) < 1e-6


def test_empty_scene_is_background():
    import paper_2601_19489_b200 as ts
    b = dict(means2d=np.zeros((0, 2)), conics=np.zeros((0, 3)), level_t=np.zeros(0),
             depths=np.zeros(0), opacities=np.zeros(0), source_ids=np.zeros(0, int),
             width=40, height=24)
    db = dev_batch(b)
    bufs = ts.render(db, ts.bin_sequential(db), np.zeros((0, 3)), (0.2, 0.4, 0.6))
    assert np.allclose(np64(bufs.color), np.array([0.2, 0.4, 0.6], np.float32))
    assert np.all(np64(bufs.final_T) == 1.0) and not np.any(np64(bufs.n_contrib))


def test_early_termination_consideration_point():
    """test_forward.py:96-107."""
    import paper_2601_19489_b200 as ts
    n = 40
    b = dev_batch(_centered(n, [0.9] * n, np.linspace(1, 2, n), sigma=40.0))
    bufs = ts.render(b, ts.bin_sequential(b), np.ones((n, 3)), np.zeros(3))
    k = int(bufs.n_considered[16, 16])
    assert k < n and float(bufs.final_T[16, 16]) < 1e-4
    assert abs(k - np.ceil(np.log(1e-4) / np.log(0.1))) <= 1


@pytest.mark.parametrize("name", ["r60", "r128", "deep"])
def test_deterministic_merge_is_bitwise_reproducible(graster, name):
    """The deterministic merge (per-pair slots summed per row in emission
    order) reproduces itself bit for bit and matches the reference like the
    atomic merge does."""
    import paper_2601_19489_b200 as ts
    from conftest import rel_err
    g = graster
    b = batch_from(g, name + "_")
    db = dev_batch(b)
    tiles = ts.bin_sequential(db)
    bufs = ts.render(db, tiles, g[name + "_colors"], g[name + "_bg"])
    args = (bufs, db, tiles, g[name + "_colors"], g[name + "_gc"], g[name + "_gd"],
            g[name + "_gt"])
    a = ts.backward_per_gaussian(*args, deterministic=True)
    c = ts.backward_per_gaussian(*args, deterministic=True)
    for k in ("d_means2d", "d_conics", "d_opacities", "d_colors", "d_depths"):
        x, y = getattr(a, k).cpu().numpy(), getattr(c, k).cpu().numpy()
        assert np.array_equal(x, y), k
        assert rel_err(x, g[f"{name}_pg_{k}"]) < 1e-4, k
    assert a.merges == int(g[name + "_merges"])


def test_blend_weights_plus_final_T_is_one():
    """test_forward.py:59-69: white splats on black, colour = sum of weights."""
    import paper_2601_19489_b200 as ts
    rng = np.random.default_rng(0)
    n = 25
    b = dict(means2d=np.stack([rng.uniform(0, 64, n), rng.uniform(0, 64, n)], 1),
             conics=np.array([[0.02, 0.005, 0.03]] * n),
             level_t=np.full(n, 2 * np.log(255 * 0.7)), depths=rng.uniform(1, 5, n),
             opacities=np.full(n, 0.7), source_ids=np.arange(n), width=64, height=64)
    db = dev_batch(b)
    bufs = ts.render(db, ts.bin_sequential(db), np.ones((n, 3)), np.zeros(3))
    assert np.abs(np64(bufs.color[:, :, 0]) + np64(bufs.final_T) - 1.0).max() < 1e-6


def test_single_splat_color_gradient_closed_form():
    """test_backward.py:53-63: with one splat and unit upstream gradient,
    dL/dc = sum over pixels of its weight = sum (1 - final_T)."""
    import paper_2601_19489_b200 as ts
    b = dev_batch(_centered(1, [0.8], [2.0], sigma=5.0))
    colors = np.array([[0.3, 0.6, 0.9]])
    tiles = ts.bin_sequential(b)
    bufs = ts.render(b, tiles, colors, np.zeros(3))
    g = ts.backward_per_gaussian(bufs, b, tiles, colors, np.ones((32, 32, 3)))
    expected = float((1.0 - np64(bufs.final_T)).sum())
    assert np.allclose(np64(g.d_colors)[0], expected, rtol=1e-5)
