"""Loss contract of the reference's tests/test_losses.py through the device
losses: identity images, the (1-lam) L1 + lam (1-SSIM) combination, the
disparity loss (identity, single pixel, zero weight / empty mask, gradient,
power-of-two rescaling), the depth-weight schedule and PSNR values."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_identity_images_give_zero_loss():
    from paper_2601_19489_b200.losses import photometric
    img = np.random.default_rng(0).uniform(0, 1, (24, 24, 3))
    report, grad = photometric(img, img.copy(), 0.2)
    assert report.l1 == 0.0
    assert report.ssim == pytest.approx(1.0, abs=1e-6)
    assert abs(report.photometric) < 1e-6
    assert float(grad.abs().max()) < 1e-7


def test_photometric_is_the_combination():
    from paper_2601_19489_b200.losses import photometric
    rng = np.random.default_rng(0)
    a, b = rng.uniform(0, 1, (16, 16, 3)), rng.uniform(0, 1, (16, 16, 3))
    report, _ = photometric(a, b, 0.2)
    assert report.photometric > 1e-6 and -1.0 <= report.ssim <= 1.0
    assert report.photometric == pytest.approx(0.8 * report.l1 + 0.2 * (1 - report.ssim),
                                               abs=1e-6)


def test_disparity_identity_and_single_pixel():
    from paper_2601_19489_b200.losses import disparity_loss
    d = np.full((4, 4), 2.0)
    loss, _ = disparity_loss(d, d.copy(), np.ones((4, 4), bool), 1.0)
    assert loss == 0.0
    loss, _ = disparity_loss(np.array([[1.0]]), np.array([[2.0]]), np.ones((1, 1), bool), 1.0)
    assert loss == pytest.approx(0.5)


def test_disparity_weight_zero_and_empty_mask():
    from paper_2601_19489_b200.losses import disparity_loss
    rng = np.random.default_rng(1)
    d_r, d_p = rng.uniform(0.5, 3, (8, 8)), rng.uniform(0.5, 3, (8, 8))
    for mask, w in ((np.ones((8, 8), bool), 0.0), (np.zeros((8, 8), bool), 1.0)):
        loss, grad = disparity_loss(d_r, d_p, mask, w)
        assert loss == 0.0 and not bool(grad.any())


def test_disparity_gradient_matches_analytic_float64():
    """d/d d_r of w mean_valid |1/d_r - 1/d_p| = -w sign(diff) / (n d_r^2)."""
    from paper_2601_19489_b200.losses import disparity_loss
    rng = np.random.default_rng(2)
    d_r = np.asarray(rng.uniform(0.5, 3.0, (8, 8)), np.float32).astype(np.float64)
    d_p = np.asarray(rng.uniform(0.5, 3.0, (8, 8)), np.float32).astype(np.float64)
    mask = rng.uniform(0, 1, (8, 8)) > 0.3
    loss, grad = disparity_loss(d_r, d_p, mask, 0.7)
    diff = 1 / d_r - 1 / d_p
    ref = np.where(mask, -0.7 * np.sign(diff) / (mask.sum() * d_r ** 2), 0.0)
    assert float(loss) == pytest.approx(0.7 * np.abs(diff[mask]).mean(), rel=1e-5)
    got = grad.cpu().numpy()
    assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-5


@pytest.mark.parametrize("log2_k", [-3, 0, 2, 6])
def test_disparity_power_of_two_rescaling(log2_k):
    """loss(k d_r, k d_p) == loss(d_r, d_p) / k for power-of-two k."""
    from paper_2601_19489_b200.losses import disparity_loss
    k = float(2.0 ** log2_k)
    rng = np.random.default_rng(7)
    d_r = np.asarray(rng.uniform(0.5, 4.0, (6, 6)), np.float32).astype(np.float64)
    d_p = np.asarray(rng.uniform(0.5, 4.0, (6, 6)), np.float32).astype(np.float64)
    mask = np.ones((6, 6), bool)
    base, _ = disparity_loss(d_r, d_p, mask, 1.0)
    scaled, _ = disparity_loss(k * d_r, k * d_p, mask, 1.0)
    assert float(scaled) == pytest.approx(float(base) / k, rel=1e-6)


def test_depth_weight_schedule():
    from paper_2601_19489_b200.losses import depth_weight_schedule
    assert depth_weight_schedule(0, 1000) == pytest.approx(0.1)
    assert depth_weight_schedule(500, 1000) == 0.0
    assert depth_weight_schedule(900, 1000) == 0.0
    assert depth_weight_schedule(250, 1000) == pytest.approx(0.05)


def test_psnr_values():
    from paper_2601_19489_b200.losses import psnr
    img = np.full((4, 4, 3), 0.5)
    assert psnr(img, img.copy()) == 99.0
    assert psnr(np.zeros((10, 10, 3)), np.full((10, 10, 3), 0.1)) == pytest.approx(20.0, abs=1e-5)
    assert psnr(np.full((8, 8, 3), 0.5), np.zeros((8, 8, 3))) == pytest.approx(
        -10 * np.log10(0.25), abs=1e-5)


@pytest.mark.parametrize("with_valid", [False, True])
def test_fused_depth_chain_matches_reference_formula(with_valid):
    """csrc/depth.cu (disparity loss on D / (1 - T_f) + its chain,
    trainer.py:201-214) against the reference's float64 formula on random
    buffers with masked, empty (n_contrib = 0) and d < eps pixels."""
    import torch
    from paper_2601_19489_b200 import losses
    rng = np.random.default_rng(3)
    H, W = 67, 91
    depth = rng.uniform(0.0, 5.0, (H, W))
    final_T = rng.uniform(0.0, 0.95, (H, W))
    depth[:3] = 1e-7  # d < eps: zero gradient
    n_contrib = rng.integers(0, 4, (H, W))
    prior = rng.uniform(0.5, 8.0, (H, W))
    valid = rng.uniform(size=(H, W)) > 0.3 if with_valid else None
    w = 0.37
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    depth, final_T, prior = f32(depth), f32(final_T), f32(prior)
    mask = n_contrib > 0
    if valid is not None:
        mask &= valid
    d = np.where(mask, depth / (1.0 - final_T), 0.0)
    dr, dp = np.maximum(d, 1e-4), np.maximum(prior, 1e-4)
    diff = 1.0 / dr - 1.0 / dp
    n = mask.sum()
    ref_loss = w * np.abs(diff)[mask].mean()
    g = w * np.sign(diff) * (-1.0 / (dr * dr)) / n
    g = np.where(mask & (d >= 1e-4), g, 0.0)
    ref_gd = np.where(mask, g / (1.0 - final_T), 0.0)
    ref_gt = np.where(mask, g * depth / (1.0 - final_T) ** 2, 0.0)
    dev = lambda a, t=torch.float32: torch.as_tensor(a, dtype=t, device="cuda")  # noqa: E731
    e = dev(np.array(0.25))
    loss, gd, gt, total = losses.depth_chain_device(
        dev(depth), dev(final_T), dev(n_contrib, torch.int32), dev(prior),
        None if valid is None else dev(valid, torch.bool), w, e_photo=e)
    assert abs(float(loss) - ref_loss) <= 1e-5 * ref_loss
    assert abs(float(total) - (0.25 + ref_loss)) <= 1e-5
    for got, ref in ((gd, ref_gd), (gt, ref_gt)):
        got = got.cpu().numpy().astype(np.float64)
        assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max()
    # device weight (graph replay) and an empty mask
    loss2, *_ = losses.depth_chain_device(dev(depth), dev(final_T), dev(n_contrib * 0, torch.int32),
                                          dev(prior), None, dev(np.array(w)))
    assert float(loss2) == 0.0
