"""Vertex stage on the B200 (reference: tilesplat/projection.py).

`project` runs K1 (csrc/preprocess.cu): projection, culling, EWA conic, level
set, SH colour and the exact per-splat tile count, with rows compacted in
source order.  `project_vjp` runs K4b (csrc/vjp_adam.cu).

SplatBatch keeps the reference fields (projection.py:30-54).  On the device
they are views into one packed (M, 12) raster record so the rasterizer gathers
a splat with three 16-byte loads:
    rec[:, 0:2] means2d, rec[:, 2:5] conics, rec[:, 5] opacities,
    rec[:, 6] depths, rec[:, 7] level_t, rec[:, 8:11] per-row RGB.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .pose import PoseDelta, apply_delta, so3_left_jacobian
from .scene import Camera, GaussianSet, _device, as_device_f32

COV_DILATION = 0.3
MIN_OPACITY = 1.0 / 255.0


class SplatBatch:
    """Projected per-view state (projection.py:30-54) on the device."""

    def __init__(self, means2d, conics, level_t, depths, opacities, source_ids,
                 width, height, x_min=None, x_max=None, y_min=None, y_max=None,
                 tile_rect=None, *, _rec=None):
        self.width = int(width)
        self.height = int(height)
        if _rec is None:
            means2d = as_device_f32(means2d, (-1, 2))
            m = means2d.shape[0]
            rec = torch.zeros((m, _lib.REC_FLOATS), dtype=torch.float32, device=_device())
            rec[:, 0:2] = means2d
            rec[:, 2:5] = as_device_f32(conics, (-1, 3))
            rec[:, 5] = as_device_f32(opacities, (-1,))
            rec[:, 6] = as_device_f32(depths, (-1,))
            rec[:, 7] = as_device_f32(level_t, (-1,))
            if isinstance(source_ids, torch.Tensor):
                sid = source_ids.to(device=_device(), dtype=torch.int32)
            else:
                sid = torch.as_tensor(np.asarray(source_ids, dtype=np.int32), device=_device())
            _rec = rec
            source_ids = sid
        self.rec = _rec
        self.source_ids = source_ids
        self.x_min, self.x_max, self.y_min, self.y_max = x_min, x_max, y_min, y_max
        self.tile_rect = tile_rect
        # filled by project(): inverse map and K1's fused pair count outputs
        self.row_of_source = None
        self.counts = None       # (M,) int32 pairs per row
        self.depth_bits = None   # (M,) int32 view of the f32 depth bits
        self.spans = None        # (M, 4) int32 compact column walk
        self.totals = None       # (2,) int64 device [M, P]
        self.n_pairs = None
        self.strategy = None

    # reference field names as views into the packed record
    @property
    def means2d(self):
        return self.rec[:, 0:2]

    @property
    def conics(self):
        return self.rec[:, 2:5]

    @property
    def opacities(self):
        return self.rec[:, 5]

    @property
    def depths(self):
        return self.rec[:, 6]

    @property
    def level_t(self):
        return self.rec[:, 7]

    @property
    def colors(self):
        """Per-row RGB written by project() (trainer._splat_colors)."""
        return self.rec[:, 8:11]

    def __len__(self):
        return self.rec.shape[0]


@dataclass
class Grad3D:
    positions: torch.Tensor
    log_scales: torch.Tensor
    rotations: torch.Tensor
    opacity_logits: torch.Tensor


@dataclass
class PoseGrad:
    rot_vec: np.ndarray = field(default_factory=lambda: np.zeros(3))
    trans: np.ndarray = field(default_factory=lambda: np.zeros(3))


def camera_struct(camera: Camera, delta: PoseDelta | None, near: float) -> _lib.Camera_t:
    R, t = apply_delta(camera, delta)
    center = -R.T @ t
    c = _lib.Camera_t()
    c.fx, c.fy, c.cx, c.cy = camera.fx, camera.fy, camera.cx, camera.cy
    c.width, c.height = camera.width, camera.height
    c.R[:] = [float(v) for v in R.reshape(-1)]
    c.t[:] = [float(v) for v in t]
    c.center[:] = [float(v) for v in center]
    c.near_plane = near
    return c


def gaussians_struct(gset: GaussianSet) -> _lib.Gaussians_t:
    g = _lib.Gaussians_t()
    g.positions = gset.positions.data_ptr()
    g.log_scales = gset.log_scales.data_ptr()
    g.rotations = gset.rotations.data_ptr()
    g.opacity_logits = gset.opacity_logits.data_ptr()
    g.colors = gset.colors.data_ptr()
    g.n = len(gset)
    g.sh_coeffs = gset.colors.shape[1]
    return g


class ProjectionScratch:
    """Capacity buffers for K1 (reused across views of the same set size)."""

    def __init__(self, n: int):
        dev = _device()
        lib = _lib.load()
        self.n = n
        self.rec = torch.empty((max(n, 1), _lib.REC_FLOATS), dtype=torch.float32, device=dev)
        self.source_ids = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.row_of_source = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.counts = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.depth_bits = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.spans = torch.empty((max(n, 1), 4), dtype=torch.int32, device=dev)
        self.totals = torch.zeros(2, dtype=torch.int64, device=dev)
        self.ws_bytes = int(lib.tsr_preprocess_workspace(n))
        self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)


def project_raw(gset: GaussianSet, camera: Camera, near: float, delta, strategy: int,
                scratch: ProjectionScratch | None = None) -> ProjectionScratch:
    """Launch K1 without any host synchronisation."""
    lib = _lib.load()
    n = len(gset)
    if scratch is None or scratch.n != n:
        scratch = ProjectionScratch(n)
    g = gaussians_struct(gset)
    cam = camera_struct(camera, delta, near)
    _lib.check(lib.tsr_preprocess_fwd(
        g, cam, strategy, scratch.rec.data_ptr(), scratch.source_ids.data_ptr(),
        scratch.row_of_source.data_ptr(), scratch.counts.data_ptr(),
        scratch.depth_bits.data_ptr(), scratch.spans.data_ptr(), scratch.totals.data_ptr(),
        scratch.workspace.data_ptr(), scratch.ws_bytes, _lib.stream_handle()),
        "tsr_preprocess_fwd")
    return scratch


def batch_from_scratch(scratch: ProjectionScratch, camera: Camera, strategy: int) -> SplatBatch:
    m, p = (int(v) for v in scratch.totals.tolist())
    batch = SplatBatch(None, None, None, None, None, scratch.source_ids[:m],
                       camera.width, camera.height, _rec=scratch.rec[:m])
    attach_counts(batch, scratch, m, p, strategy)
    return batch


def attach_counts(batch: SplatBatch, scratch, m: int, p: int, strategy: int) -> None:
    batch.row_of_source = scratch.row_of_source[: scratch.n]
    batch.counts = scratch.counts[:m]
    batch.depth_bits = scratch.depth_bits[:m]
    batch.spans = scratch.spans[:m]
    batch.totals = scratch.totals
    batch.n_pairs = p
    batch.strategy = strategy


def project(gset: GaussianSet, camera: Camera, near: float = 0.01,
            delta: PoseDelta | None = None, *, strategy: int = 0) -> SplatBatch:
    """K1: cull + EWA projection + colour + exact tile count (projection.py:112-136).
    Output rows preserve source order."""
    scratch = project_raw(gset, camera, near, delta, strategy)
    return batch_from_scratch(scratch, camera, strategy)


def _pose_grad_from_sums(sums: np.ndarray, camera: Camera, delta) -> PoseGrad:
    """Finish the pose chain on the host from the 12 reduced sums
    (projection.py:232-240)."""
    S1 = sums[:9].reshape(3, 3)
    S2 = sums[9:12]
    out = PoseGrad()
    out.trans = camera.rotation.T @ S2
    G_Rdelta = camera.rotation.T @ S1
    R_delta = delta.rotation() if delta is not None else np.eye(3)
    B = R_delta @ G_Rdelta.T
    g_omega = np.array([B[1, 2] - B[2, 1], B[2, 0] - B[0, 2], B[0, 1] - B[1, 0]])
    rot_vec = delta.rot_vec if delta is not None else np.zeros(3)
    out.rot_vec = so3_left_jacobian(rot_vec).T @ g_omega
    return out


def project_vjp(gset: GaussianSet, camera: Camera, batch: SplatBatch, grads2d,
                near: float = 0.01, delta: PoseDelta | None = None, *,
                grad_colors: torch.Tensor | None = None, with_pose: bool = True):
    """K4b: 2D splat gradients -> 3D parameters and pose (projection.py:139-241).

    `grads2d` is a Grad2D (packed) or any object with d_means2d, d_conics,
    d_depths, d_opacities (and optionally d_colors).  Returns (Grad3D, PoseGrad);
    when `grad_colors` (N,C,3) is given it receives the colour/SH gradient
    (trainer._full_grads)."""
    from .backward import Grad2D
    lib = _lib.load()
    n = len(gset)
    # culling must match (projection.py:147-150): re-run K1 into scratch
    check = project_raw(gset, camera, near, delta, 0)
    m_check = int(check.totals[0].item())
    if m_check != len(batch) or not torch.equal(check.source_ids[:m_check],
                                                 batch.source_ids.to(torch.int32)):
        raise ValueError("batch does not match projection inputs (culling differs)")
    row_of_source = check.row_of_source
    packed = grads2d.packed if isinstance(grads2d, Grad2D) else Grad2D.pack(grads2d, len(batch))
    dev = _device()
    grad = Grad3D(torch.empty((n, 3), device=dev), torch.empty((n, 3), device=dev),
                  torch.empty((n, 4), device=dev), torch.empty((n,), device=dev))
    gcol = grad_colors if grad_colors is not None else torch.empty_like(gset.colors)
    pose_sums = torch.zeros(12, dtype=torch.float32, device=dev) if with_pose else None
    _lib.check(lib.tsr_preprocess_bwd(
        gaussians_struct(gset), camera_struct(camera, delta, near), batch.rec.data_ptr(),
        row_of_source.data_ptr(), packed.data_ptr(), grad.positions.data_ptr(),
        grad.log_scales.data_ptr(), grad.rotations.data_ptr(), grad.opacity_logits.data_ptr(),
        gcol.data_ptr(), _lib.ptr(pose_sums), 0, _lib.stream_handle()), "tsr_preprocess_bwd")
    pose = PoseGrad()
    if with_pose:
        pose = _pose_grad_from_sums(pose_sums.double().cpu().numpy(), camera, delta)
    return grad, pose
