"""SURVEY.md §8(f) #2-#4 parity: K3 scoring mode, density scores and
decisions, optimiser resize, PLY files and the training loop, against the
unmodified reference's golden vectors (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from conftest import GOLDEN, batch_from, dev_batch, golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gd():
    return golden("density")


def _scored(gd, v):
    import paper_2601_19489_b200 as ts
    b = batch_from(gd, f"v{v}_")
    db = dev_batch(b)
    tiles = ts.bin_sequential(db)
    bufs, con = ts.render(db, tiles, gd[f"v{v}_colors"], np.zeros(3), scoring=True)
    return db, tiles, bufs, con


@pytest.mark.parametrize("v", [0, 1])
def test_contributions_multiset_matches_reference(gd, v):
    _, _, bufs, con = _scored(gd, v)
    got = np.stack([con.pixel_idx.cpu().numpy(), con.splat_rows.cpu().numpy()], 1)
    ref = np.stack([gd[f"v{v}_pix"], gd[f"v{v}_rows"]], 1)
    assert got.shape == ref.shape
    assert np.array_equal(got[np.lexsort(got.T[::-1])], ref[np.lexsort(ref.T[::-1])])
    assert np.abs(bufs.color.cpu().numpy() - gd[f"v{v}_color"]).max() < 2e-5


@pytest.mark.parametrize("v", [0, 1])
def test_error_mask_matches_reference(gd, v):
    import paper_2601_19489_b200 as ts
    m = ts.error_mask(gd[f"v{v}_color"], gd[f"v{v}_gt"], 0.5)
    assert np.array_equal(m.mask.cpu().numpy(), gd[f"v{v}_mask"])
    assert np.abs(m.e.cpu().numpy() - gd[f"v{v}_e"]).max() < 1e-12


def test_scores_match_reference(gd):
    import paper_2601_19489_b200 as ts
    masks, pix, ids, e = [], [], [], []
    for v in (0, 1):
        db, _, _, con = _scored(gd, v)
        masks.append(ts.error_mask(gd[f"v{v}_color"], gd[f"v{v}_gt"], 0.5))
        pix.append(con.pixel_idx)
        ids.append(db.source_ids[con.splat_rows])
        e.append(float(gd[f"v{v}_ephoto"]))
    sp = ts.score_densify(masks, pix, ids, 90).cpu().numpy()
    sm = ts.score_prune(masks, pix, ids, e, 90).cpu().numpy()
    assert np.array_equal(sp, gd["s_plus"])
    assert np.abs(sm - gd["s_minus"]).max() < 1e-12


def test_fused_masked_counts_equal_contribution_bincount(gd):
    """K3 mode 3 (the trainer's path) == bincount of the masked lists."""
    import torch
    import paper_2601_19489_b200 as ts
    from paper_2601_19489_b200.density import masked_row_counts
    for v in (0, 1):
        db, tiles, _, con = _scored(gd, v)
        m = ts.error_mask(gd[f"v{v}_color"], gd[f"v{v}_gt"], 0.5)
        fused = masked_row_counts(db, tiles, np.zeros(3), m)
        hits = m.mask.reshape(-1)[con.pixel_idx]
        ref = torch.bincount(con.splat_rows[hits], minlength=len(db)).float()
        assert torch.equal(fused, ref)


@pytest.mark.parametrize("case", ["dec", "floor"])
def test_apply_decisions_match_reference(gd, case):
    import paper_2601_19489_b200 as ts
    params = {k[4:]: v for k, v in gd.items() if k.startswith("set_")}
    gset = ts.GaussianSet(**params)
    new, dec = ts.apply_decisions(gset, gd["dec_sp"], gd["dec_sm"], 16.0, 0.9, 0.01,
                                  np.random.default_rng(5),
                                  min_splats=16 if case == "dec" else 190)
    assert np.array_equal(dec.codes.cpu().numpy(), gd[f"{case}_actions"])
    assert len(dec) == 200 and dec[3].action in ("keep", "clone", "split", "prune")
    for k in ("positions", "log_scales", "rotations", "opacity_logits", "colors"):
        got = getattr(new, k).cpu().numpy().astype(np.float64)
        ref = np.asarray(gd[f"{case}_new_{k}"], np.float32).astype(np.float64)
        assert got.shape == ref.reshape(got.shape).shape
        assert np.abs(got - ref.reshape(got.shape)).max() <= 1e-6 * max(1.0, np.abs(ref).max())


def test_adam_resize_matches_reference(gd):
    import torch
    import paper_2601_19489_b200 as ts
    params = {k[4:]: v for k, v in gd.items() if k.startswith("set_")}
    gset = ts.GaussianSet(**params)
    _, dec = ts.apply_decisions(gset, gd["dec_sp"], gd["dec_sm"], 16.0, 0.9, 0.01,
                                np.random.default_rng(5), min_splats=16)
    opt = ts.Adam()
    p = gset.params()
    g = {k: torch.zeros_like(v) for k, v in p.items()}
    g["positions"] = torch.as_tensor(gd["adam_g_pos"], dtype=torch.float32, device="cuda")
    g["log_scales"] = torch.as_tensor(gd["adam_g_ls"], dtype=torch.float32, device="cuda")
    opt.step(p, g)
    assert np.abs(opt.moments("positions")[0].cpu().numpy() - gd["adam_m_before"]).max() < 1e-6
    opt.resize(dec)
    m_after = opt.moments("positions")[0].cpu().numpy()
    assert m_after.shape == gd["adam_m_after"].shape
    assert np.abs(m_after - gd["adam_m_after"]).max() < 1e-6
    assert np.abs(opt.moments("log_scales")[1].cpu().numpy() - gd["adam_v_after"]).max() < 1e-9


def test_ply_reference_file_round_trip(tmp_path):
    import paper_2601_19489_b200 as ts
    ref = golden("ply")
    g = ts.read_ply(GOLDEN / "ref_sh1.ply")
    h = g.to_numpy()
    for k in ("positions", "log_scales", "rotations", "opacity_logits", "colors"):
        assert np.array_equal(h[k], ref[k].reshape(h[k].shape))
    out = tmp_path / "ours.ply"
    ts.write_ply(g, out)
    assert out.read_bytes() == (GOLDEN / "ref_sh1.ply").read_bytes()  # drop-in byte format
    again = ts.read_ply(out).to_numpy()
    for k in h:
        assert np.array_equal(again[k], h[k])


def test_ply_schema_errors(tmp_path):
    import paper_2601_19489_b200 as ts
    bad = tmp_path / "bad.ply"
    bad.write_bytes(b"not a ply\n")
    with pytest.raises(ts.PlySchemaError):
        ts.read_ply(bad)
    bad.write_bytes(b"ply\nformat ascii 1.0\nend_header\n")
    with pytest.raises(ts.PlySchemaError):
        ts.read_ply(bad)


def test_train_loop_densifies_and_improves(tmp_path):
    """The reference's ablation-style scene (test_acceptance.py:427-440):
    training improves PSNR, densify rounds run through the fused scoring
    pass, the PLY and CSV outputs are written."""
    import paper_2601_19489_b200 as ts
    from paper_2601_19489_b200.synthetic import synthetic_scene
    scene, gt = synthetic_scene(n_splats=48, n_views=7, width=48, height=48, seed=21,
                                arc_degrees=70.0)
    rng = np.random.default_rng(22)
    keep = np.sort(rng.choice(48, size=26, replace=False))
    h = gt.to_numpy()
    init = {k: v[keep].copy() for k, v in h.items()}
    radial = 1.0 + rng.normal(0, 0.10, (26, 1))
    init["positions"] = init["positions"] * radial + rng.normal(0, 0.02, (26, 3))
    init["log_scales"] += rng.normal(0, 0.15, (26, 3)) + 0.15
    init["colors"] += rng.normal(0, 0.05, init["colors"].shape)
    init = ts.GaussianSet(**init)
    cfg = ts.TrainConfig(round_profile="round2", max_iters=600, budget_seconds=300.0,
                         eval_interval=100, seed=0, densify_start=100, densify_end=500,
                         densify_interval=200, consistency_views=6, theta_plus=8.0,
                         theta_minus=0.95, scale_split_threshold_frac=0.08, min_splats=8,
                         holdout_views=(3,))
    before = ts.evaluate(init, [scene.cameras[3]], cfg)
    res = ts.train(scene, cfg, initial=init, ply_path=tmp_path / "out.ply",
                   metrics_path=tmp_path / "m.csv", decisions_path=tmp_path / "d.csv")
    assert res.stop_reason == "completed" and res.iterations == 600
    psnrs = [r["psnr"] for r in res.metrics if not np.isnan(r["psnr"])]
    assert len(psnrs) == 6 and psnrs[-1] > before + 3.0
    assert all(np.isfinite(r["total"]) for r in res.metrics)
    assert (tmp_path / "d.csv").read_text().count("\n") == 1 + 2  # rounds at 200, 400
    assert len(ts.read_ply(tmp_path / "out.ply")) == len(res.gset)


def test_fused_and_reference_form_densify_scores_agree():
    import paper_2601_19489_b200 as ts
    from paper_2601_19489_b200.synthetic import synthetic_scene
    from paper_2601_19489_b200.trainer import _densify_round, _densify_round_fused
    from paper_2601_19489_b200.scene import as_device_f32
    scene, gt = synthetic_scene(n_splats=64, n_views=6, width=64, height=48, seed=3)
    cfg = ts.TrainConfig(consistency_views=4)
    pool = np.arange(6)
    gt_dev = [as_device_f32(c.gt_image) for c in scene.cameras]
    init = gt.copy()
    init.opacity_logits.mul_(0.5)
    a = _densify_round(init, scene, cfg, None, np.random.default_rng(1), pool)
    b = _densify_round_fused(init, scene, cfg, None, np.random.default_rng(1), pool, gt_dev)
    assert np.abs(a[0].cpu().numpy() - b[0].cpu().numpy()).max() == 0.0
    assert np.abs(a[1].cpu().numpy() - b[1].cpu().numpy()).max() < 1e-6
