"""Photometric / depth objectives with analytic gradients (reference:
tilesplat/losses.py).

The photometric objective E = (1 - lam) mean|r - g| + lam (1 - SSIM) and its
gradient run in one fused CUDA pipeline (csrc/loss.cu):
11-tap sigma=1.5 Gaussian window, zero padding, C1 = 0.01^2, C2 = 0.03^2
(losses.py:17-91).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .scene import as_device_f32

SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2
DISPARITY_EPS = 1e-4


@dataclass
class LossReport:
    l1: float
    ssim: float
    photometric: float
    depth_loss: float
    total: float
    lambda_: float
    depth_weight: float = 0.0


class PhotometricWorkspace:
    """Scratch for the fused loss (planar SSIM backward sources + partials)."""

    def __init__(self):
        self.buf = None
        self.key = None

    def get(self, h: int, w: int, device) -> torch.Tensor:
        if self.key != (h, w, device):
            n = int(_lib.load().tsr_photometric_workspace(h, w))
            self.buf = torch.empty(n, dtype=torch.uint8, device=device)
            self.key = (h, w, device)
        return self.buf


_default_ws = PhotometricWorkspace()


def photometric_device(rendered: torch.Tensor, gt: torch.Tensor, lam: float = 0.2,
                       grad: torch.Tensor | None = None,
                       workspace: PhotometricWorkspace | None = None):
    """(E, l1, ssim, dE/drendered): E/l1/ssim are 0-d device tensors; no host
    synchronisation."""
    if rendered.shape != gt.shape:
        raise ValueError(f"shape mismatch: {tuple(rendered.shape)} vs {tuple(gt.shape)}")
    if not 0.0 <= lam <= 1.0:
        raise ValueError("lambda must be in [0, 1]")
    if rendered.dim() != 3 or rendered.shape[2] != 3:
        raise ValueError("images must be (H, W, 3)")
    lib = _lib.load()
    r = rendered.contiguous()
    g = gt.contiguous()
    h, w = int(r.shape[0]), int(r.shape[1])
    if grad is None:
        grad = torch.empty_like(r)
    out = torch.empty(3, dtype=torch.float32, device=r.device)
    ws = (workspace or _default_ws).get(h, w, r.device)
    _lib.check(lib.tsr_photometric(r.data_ptr(), g.data_ptr(), h, w, float(lam), grad.data_ptr(),
                                   out.data_ptr(), ws.data_ptr(), ws.numel(),
                                   _lib.stream_handle()), "tsr_photometric")
    return out[0], out[1], out[2], grad


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


class DepthChainWorkspace:
    """Scratch of the depth-chain kernels (block partials + a self-resetting
    ticket); zero-filled once."""

    def __init__(self):
        self.buf = None

    def get(self, device) -> torch.Tensor:
        if self.buf is None or self.buf.device != device:
            n = int(_lib.load().tsr_depth_chain_workspace())
            self.buf = torch.zeros(n, dtype=torch.uint8, device=device)
        return self.buf


_default_dc_ws = DepthChainWorkspace()


def depth_chain_device(depth, final_T, n_contrib, prior, valid, weight, e_photo=None,
                       workspace: DepthChainWorkspace | None = None):
    """Disparity loss + its chain through d_norm = D / (1 - T_f) (losses.py:
    94-112, trainer.py:201-214) in two sync-free kernels (csrc/depth.cu).
    weight: a float or a device scalar tensor (graph replay).  Returns
    (loss, grad_depth, grad_final_T) as device tensors; with e_photo (device
    scalar) the fourth value is e_photo + loss (the step's total), else None."""
    lib = _lib.load()
    d = as_device_f32(depth)
    h, w = int(d.shape[0]), int(d.shape[1])
    t = as_device_f32(final_T)
    nb = n_contrib.to(torch.int32).contiguous()
    p = as_device_f32(prior)
    v = None
    if valid is not None:
        v = valid if isinstance(valid, torch.Tensor) else torch.as_tensor(np.asarray(valid))
        v = v.to(d.device).bool().contiguous()
    w_dev = weight if isinstance(weight, torch.Tensor) else None
    out = torch.empty(2, dtype=torch.float32, device=d.device)
    gd = torch.empty_like(d)
    gt = torch.empty_like(d)
    ws = (workspace or _default_dc_ws).get(d.device)
    _lib.check(lib.tsr_depth_chain(
        d.data_ptr(), t.data_ptr(), nb.data_ptr(), p.data_ptr(), _lib.ptr(v), h, w,
        0.0 if w_dev is not None else float(weight), _lib.ptr(w_dev),
        _lib.ptr(e_photo), out[0].data_ptr(), out[1].data_ptr(), gd.data_ptr(), gt.data_ptr(),
        ws.data_ptr(), ws.numel(), _lib.stream_handle()), "tsr_depth_chain")
    return out[0], gd, gt, (out[1] if e_photo is not None else None)


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
