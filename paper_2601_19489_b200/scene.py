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

    def replace_pose(self, rotation, translation) -> None:
        self.rotation = np.asarray(rotation, dtype=np.float64).reshape(3, 3)
        self.translation = np.asarray(translation, dtype=np.float64).reshape(3)
