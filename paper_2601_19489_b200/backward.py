"""Per-Gaussian raster backward on the B200 (reference: tilesplat/backward.py).

`backward_per_gaussian` launches K4 (csrc/backward.cu).  Grad2D keeps the
reference's fields (backward.py:36-50) as views into one packed (M, 10)
buffer {d_mx, d_my, d_a, d_b, d_c, d_opacity, d_r, d_g, d_b, d_depth} that
K4 merges into with one atomic per (splat, tile, field).  `merges` follows
the reference's count: every (splat, tile) pair of every tile whose upstream
gradient is not all zero (backward.py:214-222).
"""

from __future__ import annotations

import torch

from . import _lib
from .binning import TileIndex
from .forward import CHECKPOINT_INTERVAL, RenderBuffers, _ensure_colors
from .projection import SplatBatch
from .scene import _device, as_device_f32


class CheckpointsMissingError(RuntimeError):
    """Per-Gaussian backward needs a forward pass run with checkpointing."""


class Grad2D:
    def __init__(self, packed: torch.Tensor, merges: int = 0):
        self.packed = packed
        self.merges = merges

    @classmethod
    def zeros(cls, n: int) -> "Grad2D":
        return cls(torch.zeros((n, _lib.GRAD2D_FLOATS), dtype=torch.float32, device=_device()))

    @staticmethod
    def pack(obj, n: int) -> torch.Tensor:
        p = torch.zeros((n, _lib.GRAD2D_FLOATS), dtype=torch.float32, device=_device())
        p[:, 0:2] = as_device_f32(obj.d_means2d, (-1, 2))
        p[:, 2:5] = as_device_f32(obj.d_conics, (-1, 3))
        p[:, 5] = as_device_f32(obj.d_opacities, (-1,))
        if getattr(obj, "d_colors", None) is not None:
            p[:, 6:9] = as_device_f32(obj.d_colors, (-1, 3))
        p[:, 9] = as_device_f32(obj.d_depths, (-1,))
        return p

    @property
    def d_means2d(self):
        return self.packed[:, 0:2]

    @property
    def d_conics(self):
        return self.packed[:, 2:5]

    @property
    def d_opacities(self):
        return self.packed[:, 5]

    @property
    def d_colors(self):
        return self.packed[:, 6:9]

    @property
    def d_depths(self):
        return self.packed[:, 9]


def backward_per_gaussian_raw(buffers: RenderBuffers, batch: SplatBatch, tiles: TileIndex,
                              grad_color, grad_depth=None, grad_final_T=None,
                              out: torch.Tensor | None = None,
                              merges: torch.Tensor | None = None) -> tuple:
    """Launch K4 without host synchronisation; returns (packed grads, merges)."""
    lib = _lib.load()
    dev = _device()
    if out is None:
        out = torch.zeros((len(batch), _lib.GRAD2D_FLOATS), dtype=torch.float32, device=dev)
    if merges is None:
        merges = torch.zeros(1, dtype=torch.int64, device=dev)
    gc = as_device_f32(grad_color)
    gd = as_device_f32(grad_depth) if grad_depth is not None else None
    gt = as_device_f32(grad_final_T) if grad_final_T is not None else None
    _lib.check(lib.tsr_render_bwd(
        batch.rec.data_ptr(), _lib.ptr(tiles.values) if tiles.n_pairs else None,
        tiles.offsets.data_ptr(), batch.width, batch.height, buffers.color.data_ptr(),
        buffers.depth.data_ptr(), buffers.final_T.data_ptr(), buffers.n_considered.data_ptr(),
        _lib.ptr(buffers.ckpt), _lib.ptr(buffers.ckpt_base), gc.data_ptr(), _lib.ptr(gd),
        _lib.ptr(gt), out.data_ptr(), merges.data_ptr(), _lib.stream_handle()),
        "tsr_render_bwd")
    return out, merges


def backward_det_raw(buffers: RenderBuffers, batch: SplatBatch, tiles: TileIndex, grad_color,
                     grad_depth, grad_final_T, out: torch.Tensor, merges: torch.Tensor,
                     slots: torch.Tensor, processed: torch.Tensor, m_dev=None) -> None:
    """K4 with the deterministic merge (per-pair slots, per-row emission-order
    sums through K2's inverse permutation)."""
    lib = _lib.load()
    if tiles.det is None:
        raise ValueError("the deterministic merge needs a TileIndex built with its "
                         "permutation outputs (IndexBuffers(det=True))")
    gc = as_device_f32(grad_color)
    gd = as_device_f32(grad_depth) if grad_depth is not None else None
    gt = as_device_f32(grad_final_T) if grad_final_T is not None else None
    inv_perm, rank_row, rank_count, rank_off = tiles.det
    _lib.check(lib.tsr_render_bwd_det(
        batch.rec.data_ptr(), _lib.ptr(tiles.values) if tiles.n_pairs else None,
        tiles.offsets.data_ptr(), batch.width, batch.height, buffers.color.data_ptr(),
        buffers.depth.data_ptr(), buffers.final_T.data_ptr(), buffers.n_considered.data_ptr(),
        _lib.ptr(buffers.ckpt), _lib.ptr(buffers.ckpt_base), gc.data_ptr(), _lib.ptr(gd),
        _lib.ptr(gt), merges.data_ptr(), slots.data_ptr(), processed.data_ptr(),
        inv_perm.data_ptr(), rank_row.data_ptr(), rank_count.data_ptr(), rank_off.data_ptr(),
        tiles.keys.data_ptr(), out.shape[0], _lib.ptr(m_dev), out.data_ptr(),
        _lib.stream_handle()), "tsr_render_bwd_det")


def backward_per_gaussian(buffers: RenderBuffers, batch: SplatBatch, tiles: TileIndex,
                          colors, grad_color, grad_depth=None, grad_final_T=None,
                          group_size: int = CHECKPOINT_INTERVAL,
                          deterministic: bool = False) -> Grad2D:
    """K4 (backward.py:137-223).  deterministic=True merges through per-pair
    slots summed per row in emission order: bitwise reproducible run to run
    (the default atomic merge agrees within FP32 rounding)."""
    if group_size != CHECKPOINT_INTERVAL:
        raise ValueError("groups are one 32-lane warp (CHECKPOINT_INTERVAL)")
    if not buffers.has_checkpoints and tiles.n_pairs > group_size:
        counts = tiles.offsets[1:] - tiles.offsets[:-1]
        worst = int(counts.max().item())
        if worst > group_size:
            tile = int(torch.argmax(counts).item())
            raise CheckpointsMissingError(
                f"tile {tile} has {worst} splats but no stored checkpoints; "
                "rerun the forward pass with checkpointing enabled")
    _ensure_colors(batch, colors)
    if deterministic:
        dev = _device()
        packed = torch.empty((len(batch), _lib.GRAD2D_FLOATS), dtype=torch.float32, device=dev)
        merges = torch.zeros(1, dtype=torch.int64, device=dev)
        slots = torch.empty((max(tiles.n_pairs, 1), _lib.GRAD2D_FLOATS), dtype=torch.float32,
                            device=dev)
        processed = torch.zeros(tiles.n_tiles, dtype=torch.int32, device=dev)
        backward_det_raw(buffers, batch, tiles, grad_color, grad_depth, grad_final_T, packed,
                         merges, slots, processed)
        return Grad2D(packed, int(merges.item()))
    packed, merges = backward_per_gaussian_raw(buffers, batch, tiles, grad_color, grad_depth,
                                               grad_final_T)
    return Grad2D(packed, int(merges.item()))
