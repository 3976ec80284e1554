"""K1 projection / K4b VJP / K5 Adam parity against the reference's golden
vectors (test_projection.py / test_optim.py counterparts)."""

import numpy as np
import pytest

from conftest import batch_from, golden, np64, rel_err

pytestmark = pytest.mark.gpu

PROJ_RTOL = 2e-5     # FP32 projection of FP32-exact inputs vs float64
VJP_RTOL = 2e-4      # FP32 chain rule, max-normalised
ADAM_RTOL = 1e-5


def _camera(ts, g, prefix=""):
    f = g[prefix + "cam_f"]
    return ts.Camera(float(f[0]), float(f[1]), float(f[2]), float(f[3]), int(f[4]), int(f[5]),
                     g[prefix + "cam_R"], g[prefix + "cam_t"])


def test_project_and_vjp_match_reference():
    import paper_2601_19489_b200 as ts
    g = golden("projection")
    params = {k[2:]: v for k, v in g.items() if k.startswith("p_")}
    gset = ts.GaussianSet(**params)
    cam = _camera(ts, g)
    batch = ts.project(gset, cam, near=0.1)
    ref = batch_from(g, "b_")
    assert np.array_equal(np64(batch.source_ids), ref["source_ids"])
    for k in ("means2d", "conics", "level_t", "depths", "opacities"):
        assert rel_err(np64(getattr(batch, k)), ref[k]) < PROJ_RTOL, k

    class G:
        pass

    g2 = G()
    g2.d_means2d, g2.d_conics = g["g_means"], g["g_conics"]
    g2.d_depths, g2.d_opacities = g["g_depths"], g["g_opac"]
    g3, pose = ts.project_vjp(gset, cam, batch, g2, near=0.1)
    for k in ("positions", "log_scales", "rotations", "opacity_logits"):
        assert rel_err(np64(getattr(g3, k)), g[f"g3_{k}"]) < VJP_RTOL, k
    assert rel_err(np.concatenate([pose.rot_vec, pose.trans]), g["pose"]) < VJP_RTOL


def test_vjp_rejects_mismatched_batch():
    import paper_2601_19489_b200 as ts
    g = golden("projection")
    params = {k[2:]: v for k, v in g.items() if k.startswith("p_")}
    gset = ts.GaussianSet(**params)
    cam = _camera(ts, g)
    batch = ts.project(gset, cam, near=0.1)
    batch.source_ids = batch.source_ids[:-1]
    batch.rec = batch.rec[:-1]
    with pytest.raises(ValueError, match="culling"):
        ts.project_vjp(gset, cam, batch, ts.Grad2D.zeros(len(batch)), near=0.1)


def test_adam_matches_reference_sequence():
    import torch
    import paper_2601_19489_b200 as ts
    g = golden("adam")
    names = ("positions", "rotations", "colors")
    opt = ts.Adam({"positions": 1e-2, "rotations": 0.1, "colors": 3e-3})
    p = {k: torch.tensor(g[f"init_{k}"], dtype=torch.float32, device="cuda") for k in names}
    for step in range(4):
        grads = {k: torch.tensor(g[f"g{step}_{k}"], dtype=torch.float32, device="cuda")
                 for k in names}
        skipped = opt.step(p, grads)
        assert skipped == int(g[f"skipped{step}"])
        for k in names:
            assert rel_err(np64(p[k]), g[f"p{step}_{k}"]) < ADAM_RTOL, (step, k)
            m, v = opt.moments(k)
            assert rel_err(np64(m), g[f"m{step}_{k}"]) < ADAM_RTOL, (step, k)
    assert opt.skipped_rows == sum(int(g[f"skipped{s}"]) for s in range(4))


def test_adam_first_step_is_minus_lr():
    import torch
    import paper_2601_19489_b200 as ts
    opt = ts.Adam({"w": 0.07})
    p = torch.ones((1, 1), device="cuda")
    opt.step({"w": p}, {"w": torch.ones((1, 1), device="cuda")})
    assert abs(float(p[0, 0]) - 0.93) < 1e-6
    assert abs(ts.position_lr(1.6e-4, 500, 1000) - 1.6e-5) < 1e-12
