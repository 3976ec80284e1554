"""Photometric / depth objectives with analytic gradients (reference:
tilesplat/losses.py).  Round-1 implementation in device torch ops (SURVEY.md
§2 row 7: on the training step, not one of the five kernels; the fused loss
kernel is §8(f) next #1).

E = (1 - lam) mean|r - g| + lam (1 - SSIM), SSIM with the 11-tap sigma=1.5
Gaussian window, zero padding, C1 = 0.01^2, C2 = 0.03^2 (losses.py:17-70).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F

from .scene import as_device_f32

SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2
DISPARITY_EPS = 1e-4

_WIN = np.exp(-((np.arange(11) - 5.0) ** 2) / (2.0 * 1.5 ** 2))
_WIN /= _WIN.sum()
_win_cache: dict = {}


def _window(device):
    key = (device.type, device.index)
    if key not in _win_cache:
        _win_cache[key] = torch.tensor(_WIN, dtype=torch.float32, device=device)
    return _win_cache[key]


@dataclass
class LossReport:
    l1: float
    ssim: float
    photometric: float
    depth_loss: float
    total: float
    lambda_: float
    depth_weight: float = 0.0


def _filter(img: torch.Tensor) -> torch.Tensor:
    """Separable zero-padded Gaussian filter over H, W of a (C, H, W) stack."""
    w = _window(img.device)
    c = img.shape[0]
    x = img.unsqueeze(0)
    x = F.conv2d(x, w.view(1, 1, 11, 1).expand(c, 1, 11, 1), padding=(5, 0), groups=c)
    x = F.conv2d(x, w.view(1, 1, 1, 11).expand(c, 1, 1, 11), padding=(0, 5), groups=c)
    return x[0]


def ssim_device(img1: torch.Tensor, img2: torch.Tensor):
    """Mean SSIM of (H, W, C) images and its gradient w.r.t. img1 (losses.py:44-70),
    as device tensors."""
    a = img1.permute(2, 0, 1)
    b = img2.permute(2, 0, 1)
    stack = torch.cat([a, b, a * a, b * b, a * b], 0)
    f = _filter(stack)
    c = a.shape[0]
    mu1, mu2, v1, v2, v12 = f[:c], f[c:2 * c], f[2 * c:3 * c], f[3 * c:4 * c], f[4 * c:]
    s1 = v1 - mu1 * mu1
    s2 = v2 - mu2 * mu2
    s12 = v12 - mu1 * mu2
    A1 = 2.0 * mu1 * mu2 + SSIM_C1
    A2 = 2.0 * s12 + SSIM_C2
    B1 = mu1 * mu1 + mu2 * mu2 + SSIM_C1
    B2 = s1 + s2 + SSIM_C2
    smap = (A1 * A2) / (B1 * B2)
    value = smap.mean()
    g = 1.0 / smap.numel()
    dA1 = g * A2 / (B1 * B2)
    dA2 = g * A1 / (B1 * B2)
    dB1 = -g * A1 * A2 / (B1 * B1 * B2)
    dB2 = -g * A1 * A2 / (B1 * B2 * B2)
    g_mu1 = 2.0 * mu2 * (dA1 - dA2) + 2.0 * mu1 * (dB1 - dB2)
    back = _filter(torch.cat([g_mu1, dB2, 2.0 * dA2], 0))
    grad = back[:c] + back[c:2 * c] * 2.0 * a + back[2 * c:] * b
    return value, grad.permute(1, 2, 0)


def photometric_device(rendered: torch.Tensor, gt: torch.Tensor, lam: float = 0.2):
    """(E, l1, ssim, dE/drendered) as device tensors; no host synchronisation."""
    if rendered.shape != gt.shape:
        raise ValueError(f"shape mismatch: {tuple(rendered.shape)} vs {tuple(gt.shape)}")
    if not 0.0 <= lam <= 1.0:
        raise ValueError("lambda must be in [0, 1]")
    diff = rendered - gt
    l1 = diff.abs().mean()
    grad_l1 = torch.sign(diff) / diff.numel()
    s, gs = ssim_device(rendered, gt)
    e = (1.0 - lam) * l1 + lam * (1.0 - s)
    grad = (1.0 - lam) * grad_l1 - lam * gs
    return e, l1, s, grad


def photometric(rendered, gt, lam: float = 0.2):
    """E_photo = (1 - lam) L1 + lam (1 - SSIM); returns (report, dE/drendered)."""
    r = as_device_f32(rendered)
    g = as_device_f32(gt)
    e, l1, s, grad = photometric_device(r, g, lam)
    vals = torch.stack([e, l1, s]).tolist()
    report = LossReport(l1=vals[1], ssim=vals[2], photometric=vals[0], depth_loss=0.0,
                        total=vals[0], lambda_=lam)
    return report, grad


def disparity_loss(rendered_depth, prior_depth, valid_mask, weight: float):
    """Weighted mean |1/d_r - 1/d_p| over valid pixels (losses.py:94-112)."""
    d = as_device_f32(rendered_depth)
    p = as_device_f32(prior_depth)
    valid = torch.as_tensor(valid_mask, device=d.device).bool() \
        if not isinstance(valid_mask, torch.Tensor) else valid_mask.to(d.device).bool()
    grad = torch.zeros_like(d)
    n_valid = int(valid.sum().item())
    if n_valid == 0 or weight == 0.0:
        return 0.0, grad
    d_r = torch.clamp(d, min=DISPARITY_EPS)
    d_p = torch.clamp(p, min=DISPARITY_EPS)
    diff = 1.0 / d_r - 1.0 / d_p
    loss = weight * float(diff.abs()[valid].mean().item())
    g = weight * torch.sign(diff) * (-1.0 / (d_r * d_r)) / n_valid
    g = torch.where(d < DISPARITY_EPS, torch.zeros_like(g), g)
    grad = torch.where(valid, g, grad)
    return loss, grad


def depth_weight_schedule(iteration: int, max_iter: int, w0: float = 0.1) -> float:
    decay_end = max_iter / 2.0
    if decay_end <= 0:
        return 0.0
    return w0 * max(0.0, 1.0 - iteration / decay_end)


def psnr(img, ref) -> float:
    a = torch.clamp(as_device_f32(img), 0.0, 1.0)
    b = torch.clamp(as_device_f32(ref), 0.0, 1.0)
    mse = float(((a - b) ** 2).mean().item())
    if mse <= 0.0:
        return 99.0
    return min(99.0, -10.0 * np.log10(mse))
