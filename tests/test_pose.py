"""Pose delta algebra on the host (reference tilesplat/pose.py; its
tests/test_pose.py cases): identity, translation and rotation actions,
bake/apply consistency, composition, exp/log round trip, the left Jacobian
against a numeric derivative of the exponential.  CPU only."""

import numpy as np
import pytest

from paper_2601_19489_b200.pose import (PoseDelta, apply_delta, bake, compose, rodrigues,
                                        so3_left_jacobian, so3_log)
from paper_2601_19489_b200.scene import Camera


@pytest.fixture
def rng():
    return np.random.default_rng(0)


def _cam(R=None, t=None):
    return Camera(30.0, 30.0, 16.0, 16.0, 32, 32, np.eye(3) if R is None else R,
                  np.zeros(3) if t is None else t)


def _world_to_cam(cam, delta, X):
    R, t = apply_delta(cam, delta)
    return X @ R.T + t


def test_zero_delta_is_identity(rng):
    cam = _cam(rodrigues(rng.normal(0, 0.3, 3)), rng.normal(0, 1, 3))
    R, t = apply_delta(cam, PoseDelta())
    assert np.array_equal(R, cam.rotation) and np.array_equal(t, cam.translation)


def test_pure_translation_shifts_world_points(rng):
    cam = _cam()
    X = rng.normal(0, 1, (5, 3))
    d = PoseDelta(np.zeros(3), np.array([0.1, -0.2, 0.3]))
    assert np.allclose(_world_to_cam(cam, d, X), X + d.trans)


def test_rotation_delta_rotates_world_points(rng):
    cam = _cam()
    X = rng.normal(0, 1, (5, 3))
    d = PoseDelta(np.array([0.0, 0.0, np.pi / 2]), np.zeros(3))
    assert np.allclose(_world_to_cam(cam, d, X), X @ rodrigues(d.rot_vec).T)


def test_bake_then_apply_is_stored_pose(rng):
    cams = [_cam(rodrigues(rng.normal(0, 0.3, 3)), rng.normal(0, 1, 3)) for _ in range(3)]
    d = PoseDelta(rng.normal(0, 0.1, 3), rng.normal(0, 0.1, 3))
    expect = [apply_delta(c, d) for c in cams]
    baked = bake(d, cams)
    assert d.is_identity() and d.steps_since_bake == 0
    assert not baked.is_identity()
    for c, (R, t) in zip(cams, expect):
        assert np.allclose(c.rotation, R, atol=1e-12) and np.allclose(c.translation, t)


def test_sequential_bakes_equal_composed_bake(rng):
    base = _cam(rodrigues(rng.normal(0, 0.3, 3)), rng.normal(0, 1, 3))
    a, b = _cam(base.rotation, base.translation), _cam(base.rotation, base.translation)
    d1 = PoseDelta(rng.normal(0, 0.1, 3), rng.normal(0, 0.1, 3))
    d2 = PoseDelta(rng.normal(0, 0.1, 3), rng.normal(0, 0.1, 3))
    b1, b2 = bake(d1.copy(), [a]), bake(d2.copy(), [a])
    bake(compose(b1, b2), [b])
    assert np.allclose(a.rotation, b.rotation, atol=1e-12)
    assert np.allclose(a.translation, b.translation, atol=1e-12)


def test_rodrigues_log_roundtrip(rng):
    for _ in range(20):
        w = rng.normal(0, 1, 3)
        w *= rng.uniform(0.0, 3.0) / np.linalg.norm(w)
        assert np.allclose(so3_log(rodrigues(w)), w, atol=1e-9)
        R = rodrigues(w)
        assert np.allclose(R @ R.T, np.eye(3), atol=1e-12)


def test_rodrigues_small_angle():
    w = np.array([1e-10, -2e-10, 3e-10])
    assert np.allclose(rodrigues(w), np.eye(3) + np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]],
                                                           [-w[1], w[0], 0]]), atol=1e-18)


def test_left_jacobian_matches_numeric_dexp(rng):
    """exp(w + e) ~ exp(J_l(w) e) exp(w) to first order."""
    for _ in range(5):
        w = rng.normal(0, 0.8, 3)
        J = so3_left_jacobian(w)
        h = 1e-6
        for k in range(3):
            e = np.zeros(3)
            e[k] = h
            num = so3_log(rodrigues(w + e) @ rodrigues(w).T) / h
            assert np.allclose(num, J[:, k], atol=1e-5)
