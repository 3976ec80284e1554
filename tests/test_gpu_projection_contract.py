"""K1 projection closed forms and invariants of the reference's
tests/test_projection.py on the device (FP32 tolerances): on-axis EWA conic,
the level set t at full and floor opacity, culling (opacity floor, z <= near),
positive-definite conics in source order, t monotone in opacity, and the
joint translation invariance of the VJP (sum_i dL/dp_i == dL/dtau)."""

import numpy as np
import pytest

from conftest import np64

pytestmark = pytest.mark.gpu


def _cam(ts, fx=100.0, fy=100.0, R=None, t=None):
    return ts.Camera(fx, fy, 32.0, 32.0, 64, 64, np.eye(3) if R is None else R,
                     np.zeros(3) if t is None else t)


def _one(ts, pos, log_scale=0.0, logit=0.0):
    return ts.GaussianSet(positions=np.array([pos], float), log_scales=np.full((1, 3), log_scale),
                          rotations=np.array([[1.0, 0, 0, 0]]),
                          opacity_logits=np.array([logit], float),
                          colors=np.full((1, 1, 3), 0.5))


def test_on_axis_isotropic_ewa():
    import paper_2601_19489_b200 as ts
    s = 0.02
    b = ts.project(_one(ts, [0, 0, 1.0], np.log(s)), _cam(ts), near=0.1)
    assert len(b) == 1
    var = (100.0 * s) ** 2 + 0.3
    a_, b_, c_ = np64(b.conics)[0]
    assert a_ == pytest.approx(1 / var, rel=1e-6) and c_ == pytest.approx(1 / var, rel=1e-6)
    assert abs(b_) < 1e-9
    assert np.allclose(np64(b.means2d)[0], [32.0, 32.0]) and float(b.depths[0]) == 1.0


def test_level_t_full_opacity_and_culling():
    import paper_2601_19489_b200 as ts
    cam = _cam(ts)
    full = ts.project(_one(ts, [0, 0, 2.0], logit=40.0), cam, near=0.1)
    assert float(full.level_t[0]) == pytest.approx(2 * np.log(255.0), rel=1e-6)
    low = np.log((1 / 300) / (1 - 1 / 300))  # opacity 1/300 < 1/255
    assert len(ts.project(_one(ts, [0, 0, 2.0], logit=low), cam, near=0.1)) == 0
    assert len(ts.project(_one(ts, [0, 0, -1.0]), cam, near=0.1)) == 0
    assert len(ts.project(_one(ts, [0, 0, 0.1]), cam, near=0.1)) == 0  # z > near, strict


def test_conics_pd_source_order_and_t_monotone():
    import paper_2601_19489_b200 as ts
    rng = np.random.default_rng(0)
    n = 40
    gset = ts.GaussianSet(positions=rng.normal(0, 0.3, (n, 3)) + [0, 0, 3.0],
                          log_scales=np.log(rng.uniform(0.02, 0.1, (n, 3))),
                          rotations=rng.normal(0, 1, (n, 4)),
                          opacity_logits=rng.uniform(-2, 2, n),
                          colors=rng.uniform(0, 1, (n, 1, 3)))
    b = ts.project(gset, _cam(ts, 55.0, 50.0), near=0.1)
    a, bb, c = np64(b.conics).T
    assert np.all(a > 0) and np.all(c > 0) and np.all(a * c - bb * bb > 0)
    assert np.all(np.diff(np64(b.source_ids)) > 0)
    assert np.all(np64(b.level_t) >= 0) and np.all(np64(b.depths) > 0.1)
    ops = np.linspace(0.01, 0.99, 25)
    ramp = ts.GaussianSet(positions=np.tile([0, 0, 2.0], (25, 1)), log_scales=np.zeros((25, 3)),
                          rotations=np.tile([1.0, 0, 0, 0], (25, 1)),
                          opacity_logits=np.log(ops / (1 - ops)),
                          colors=np.full((25, 1, 3), 0.5))
    assert np.all(np.diff(np64(ts.project(ramp, _cam(ts), near=0.1).level_t)) >= 0)


def test_joint_translation_invariance():
    """Moving the camera and every splat by one world vector leaves the 2D
    outputs fixed: at the identity delta, sum_i dL/dp_i == dL/dtau."""
    import paper_2601_19489_b200 as ts
    from paper_2601_19489_b200.pose import rodrigues
    rng = np.random.default_rng(5)
    n = 30
    gset = ts.GaussianSet(positions=rng.normal(0, 0.3, (n, 3)) + [0, 0, 3.0],
                          log_scales=np.log(rng.uniform(0.02, 0.1, (n, 3))),
                          rotations=rng.normal(0, 1, (n, 4)),
                          opacity_logits=rng.uniform(-1, 2, n),
                          colors=rng.uniform(0, 1, (n, 1, 3)))
    cam = _cam(ts, 55.0, 50.0, rodrigues([0.2, 0.1, -0.3]), np.array([0.5, -0.2, 0.8]))
    b = ts.project(gset, cam, near=0.1)
    m = len(b)

    class G:
        pass

    g2 = G()
    g2.d_means2d = rng.normal(0, 1, (m, 2))
    g2.d_conics = rng.normal(0, 1, (m, 3))
    g2.d_depths = rng.normal(0, 1, m)
    g2.d_opacities = rng.normal(0, 1, m)
    g3, gpose = ts.project_vjp(gset, cam, b, g2, near=0.1)
    s = np64(g3.positions).sum(axis=0)
    assert np.allclose(s, gpose.trans, rtol=1e-4, atol=1e-4 * np.abs(s).max())
