"""Data-model contract of the reference's tests/test_scene.py on the device
GaussianSet: activation, index errors, orthonormal rotation matrices,
validate() findings, camera checks, field-length errors, SH degree 0 and the
SH VJP against finite differences."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _simple(n=3):
    import paper_2601_19489_b200 as ts
    return ts.GaussianSet(positions=np.zeros((n, 3)), log_scales=np.zeros((n, 3)),
                          rotations=np.tile([1.0, 0, 0, 0], (n, 1)),
                          opacity_logits=np.zeros(n), colors=np.full((n, 1, 3), 0.5))


def test_activate_identity_and_range():
    import paper_2601_19489_b200 as ts
    scale, opacity, rot = ts.activate(_simple(), 0)
    assert np.allclose(scale, 1.0) and opacity == pytest.approx(0.5)
    assert np.allclose(rot, np.eye(3))
    with pytest.raises(IndexError):
        ts.activate(_simple(), 3)


def test_rotation_matrices_orthonormal():
    from paper_2601_19489_b200.scene import quat_to_rotmat
    R = quat_to_rotmat(np.random.default_rng(0).normal(0, 1, (50, 4))).double().cpu().numpy()
    assert np.abs(R @ np.transpose(R, (0, 2, 1)) - np.eye(3)).max() < 1e-5
    assert np.allclose(np.linalg.det(R), 1.0, atol=1e-5)


def test_validate_findings():
    import paper_2601_19489_b200 as ts
    assert ts.validate(_simple()) == []
    g = _simple()
    g.positions[1, 2] = float("nan")
    g.rotations[2] = 0.0
    report = ts.validate(g)
    assert any("splat 1" in r and "positions" in r for r in report)
    assert any("splat 2" in r and "quaternion" in r for r in report)


def test_camera_and_field_checks():
    import paper_2601_19489_b200 as ts
    R = np.eye(3)
    R[0, 1] = 1e-3
    with pytest.raises(ValueError, match="orthonormal"):
        ts.Camera(50, 50, 16, 16, 32, 32, R, np.zeros(3))
    cam = ts.Camera(50, 50, 20, 10, 40, 17, np.eye(3), np.zeros(3))
    assert cam.tiles_x == 3 and cam.tiles_y == 2
    with pytest.raises(ValueError, match="length"):
        ts.GaussianSet(np.zeros((3, 3)), np.zeros((2, 3)), np.tile([1.0, 0, 0, 0], (3, 1)),
                       np.zeros(3), np.zeros((3, 1, 3)))


def test_eval_sh_degree0_is_plain_rgb():
    from paper_2601_19489_b200.scene import eval_sh
    rng = np.random.default_rng(1)
    c = np.asarray(rng.uniform(0, 1, (5, 1, 3)), np.float32)
    assert np.array_equal(eval_sh(c, rng.normal(0, 1, (5, 3))).cpu().numpy(), c[:, 0, :])


@pytest.mark.parametrize("degree", [1, 2, 3])
def test_eval_sh_vjp_matches_finite_differences(degree):
    import torch
    from paper_2601_19489_b200.scene import eval_sh, eval_sh_vjp
    rng = np.random.default_rng(degree)
    n, C = 4, (degree + 1) ** 2
    coeffs = rng.normal(0, 0.5, (n, C, 3))
    dirs = rng.normal(0, 1, (n, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    gcol = rng.normal(0, 1, (n, 3))
    gc, gd = eval_sh_vjp(coeffs, dirs, gcol)
    # the VJP is linear in coefficients: exact check of d coeffs
    basis = torch.autograd.functional.jacobian(
        lambda c: eval_sh(c, dirs), torch.as_tensor(coeffs, dtype=torch.float32, device="cuda"))
    ref_c = torch.einsum("nd,ndmcq->mcq", torch.as_tensor(gcol, dtype=torch.float32,
                                                          device="cuda"), basis)
    assert torch.allclose(gc, ref_c, atol=1e-5)
    # directions: float64 central differences of the basis polynomials
    h = 1e-3
    num = np.zeros((n, 3))
    for k in range(3):
        e = np.zeros(3)
        e[k] = h
        fp = (eval_sh(coeffs, dirs + e).double().cpu().numpy() * gcol).sum(1)
        fm = (eval_sh(coeffs, dirs - e).double().cpu().numpy() * gcol).sum(1)
        num[:, k] = (fp - fm) / (2 * h)
    assert np.abs(gd.cpu().numpy() - num).max() / np.abs(num).max() < 1e-2
