"""Gaussian set and camera on the B200 (reference: tilesplat/scene.py).

`GaussianSet` keeps the reference's structure-of-arrays layout and field names
(scene.py:50-106) as FP32 CUDA tensors: positions (N,3), log_scales (N,3),
rotations (N,4) w,x,y,z, opacity_logits (N,), colors (N,C,3) SH coefficients.
`Camera` keeps the reference's pinhole + world-to-camera pose (scene.py:139-183)
on the host in float64 (a camera is 17 numbers); images live on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

TILE = 16


def _device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def as_device_f32(x, shape=None) -> torch.Tensor:
    """numpy / torch input -> contiguous FP32 tensor on the current CUDA device."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=_device(), dtype=torch.float32)
    else:
        t = torch.as_tensor(np.asarray(x, dtype=np.float32), device=_device())
    if shape is not None:
        t = t.reshape(shape)
    return t.contiguous()


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def inverse_sigmoid(y):
    return np.log(y / (1.0 - y))


@dataclass
class GaussianSet:
    positions: torch.Tensor
    log_scales: torch.Tensor
    rotations: torch.Tensor
    opacity_logits: torch.Tensor
    colors: torch.Tensor

    def __post_init__(self):
        self.positions = as_device_f32(self.positions, (-1, 3))
        self.log_scales = as_device_f32(self.log_scales, (-1, 3))
        self.rotations = as_device_f32(self.rotations, (-1, 4))
        self.opacity_logits = as_device_f32(self.opacity_logits, (-1,))
        colors = as_device_f32(self.colors)
        if colors.dim() == 2:
            colors = colors[:, None, :].contiguous()
        self.colors = colors
        n = self.positions.shape[0]
        for name in ("log_scales", "rotations", "opacity_logits", "colors"):
            if getattr(self, name).shape[0] != n:
                raise ValueError(f"field {name} has length {getattr(self, name).shape[0]}, "
                                 f"expected {n}")
        if self.colors.shape[1] not in (1, 4, 9, 16) or self.colors.shape[2] != 3:
            raise ValueError(f"colors must be (N, (deg+1)^2, 3) with deg <= 3, "
                             f"got {tuple(self.colors.shape)}")

    def __len__(self):
        return self.positions.shape[0]

    @property
    def sh_degree(self) -> int:
        return int(round(np.sqrt(self.colors.shape[1]))) - 1

    def copy(self) -> "GaussianSet":
        return GaussianSet(self.positions.clone(), self.log_scales.clone(),
                           self.rotations.clone(), self.opacity_logits.clone(),
                           self.colors.clone())

    def params(self) -> dict:
        """Optimizer groups keyed like the reference trainer (trainer.py:341-343)."""
        return {"positions": self.positions, "log_scales": self.log_scales,
                "rotations": self.rotations, "opacity_logits": self.opacity_logits,
                "colors": self.colors}

    def to_numpy(self) -> dict:
        return {k: v.detach().cpu().numpy().astype(np.float64) for k, v in self.params().items()}

    def scales(self) -> torch.Tensor:
        return torch.exp(self.log_scales)

    def opacities(self) -> torch.Tensor:
        return torch.sigmoid(self.opacity_logits)

    def rotation_matrices(self) -> torch.Tensor:
        return quat_to_rotmat(self.rotations)


def quat_normalize(quats) -> torch.Tensor:
    """Unit wxyz quaternions (scene.py:25-30); zero-norm rows stay zero."""
    q = as_device_f32(quats, (-1, 4))
    n = torch.linalg.norm(q, dim=1, keepdim=True)
    return torch.where(n > 0, q / torch.where(n > 0, n, torch.ones_like(n)), q)


def quat_to_rotmat(quats) -> torch.Tensor:
    """(N, 3, 3) rotation matrices of normalised wxyz quaternions (scene.py:33-47)."""
    w, x, y, z = quat_normalize(quats).unbind(1)
    return torch.stack([
        torch.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], 1),
        torch.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], 1),
        torch.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1),
    ], 1)


def activate(gset: GaussianSet, index: int):
    """(scale (3,), opacity, rotation (3, 3)) of one splat (scene.py:109-116)."""
    if not 0 <= index < len(gset):
        raise IndexError(f"splat index {index} out of range [0, {len(gset)})")
    scale = torch.exp(gset.log_scales[index]).cpu().numpy().astype(np.float64)
    opacity = float(torch.sigmoid(gset.opacity_logits[index]))
    rot = quat_to_rotmat(gset.rotations[index:index + 1])[0].cpu().numpy().astype(np.float64)
    return scale, opacity, rot


def validate(gset: GaussianSet) -> list:
    """Violated invariants, one line per (splat, problem); [] when clean
    (scene.py:119-137): non-finite fields, zero-norm quaternions."""
    report = []
    n = len(gset)
    for name, arr in gset.params().items():
        bad = ~torch.isfinite(arr.reshape(n, -1)).all(dim=1)
        for i in torch.nonzero(bad).flatten().tolist():
            report.append(f"splat {i}: non-finite {name}")
    norms = torch.linalg.norm(gset.rotations, dim=1)
    for i in torch.nonzero(~(norms > 0)).flatten().tolist():
        report.append(f"splat {i}: zero-norm quaternion")
    return report


# Real SH basis with the l = 0 term equal to 1 (degree 0 == plain RGB),
# scene.py:186-276; the kernels evaluate the same basis (tsr_common.cuh).
_C1 = 0.4886025119029199
_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
       0.5462742152960396)
_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
       -0.4570457994644658, 1.445305721320277, -0.5900435899266435)


def sh_basis(degree: int, dirs) -> torch.Tensor:
    """(N, (degree+1)^2) basis values at unit directions."""
    d = as_device_f32(dirs, (-1, 3))
    x, y, z = d.unbind(1)
    cols = [torch.ones_like(x)]
    if degree >= 1:
        cols += [-_C1 * y, _C1 * z, -_C1 * x]
    if degree >= 2:
        xx, yy, zz = x * x, y * y, z * z
        cols += [_C2[0] * x * y, _C2[1] * y * z, _C2[2] * (2 * zz - xx - yy), _C2[3] * x * z,
                 _C2[4] * (xx - yy)]
    if degree >= 3:
        cols += [_C3[0] * y * (3 * xx - yy), _C3[1] * x * y * z, _C3[2] * y * (4 * zz - xx - yy),
                 _C3[3] * z * (2 * zz - 3 * xx - 3 * yy), _C3[4] * x * (4 * zz - xx - yy),
                 _C3[5] * z * (xx - yy), _C3[6] * x * (xx - 3 * yy)]
    return torch.stack(cols, 1)


def eval_sh(coeffs, dirs) -> torch.Tensor:
    """View-dependent colours (N, 3) from SH coefficients (N, C, 3)."""
    c = as_device_f32(coeffs)
    degree = int(round(np.sqrt(c.shape[1]))) - 1
    if degree == 0:
        return c[:, 0, :].clone()
    return torch.einsum("nc,ncd->nd", sh_basis(degree, dirs), c)


def eval_sh_vjp(coeffs, dirs, grad_color):
    """(d coeffs, d dirs) of eval_sh for upstream grad_color (N, 3)
    (scene.py:279-291); the direction part by autograd of the basis."""
    c = as_device_f32(coeffs)
    g = as_device_f32(grad_color, (-1, 3))
    degree = int(round(np.sqrt(c.shape[1]))) - 1
    if degree == 0:
        gc = torch.zeros_like(c)
        gc[:, 0, :] = g
        return gc, torch.zeros((c.shape[0], 3), device=c.device)
    d = as_device_f32(dirs, (-1, 3)).clone().requires_grad_(True)
    with torch.enable_grad():
        basis = sh_basis(degree, d)
        out = torch.einsum("nc,ncd->nd", basis, c)
        (gd,) = torch.autograd.grad(out, d, grad_outputs=g)
    return basis.detach()[:, :, None] * g[:, None, :], gd


@dataclass
class Camera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    rotation: np.ndarray
    translation: np.ndarray
    gt_image: object = None      # (H, W, 3) in [0, 1]; numpy or tensor
    depth_prior: object = None   # (H, W)
    depth_valid: object = None   # (H, W) bool
    name: str = ""
    camera_id: int = 0

    def __post_init__(self):
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(3, 3)
        self.translation = np.asarray(self.translation, dtype=np.float64).reshape(3)
        err = np.abs(self.rotation @ self.rotation.T - np.eye(3)).max()
        if err >= 1e-5:
            raise ValueError(f"world_to_cam rotation not orthonormal (|R R^T - I|_inf = {err:.3g})")

    @property
    def tiles_x(self) -> int:
        return -(-self.width // TILE)

    @property
    def tiles_y(self) -> int:
        return -(-self.height // TILE)

    def center(self) -> np.ndarray:
        return -self.rotation.T @ self.translation

    def world_to_cam(self, points) -> np.ndarray:
        return np.asarray(points, dtype=np.float64) @ self.rotation.T + self.translation

    def replace_pose(self, rotation, translation) -> None:
        self.rotation = np.asarray(rotation, dtype=np.float64).reshape(3, 3)
        self.translation = np.asarray(translation, dtype=np.float64).reshape(3)
