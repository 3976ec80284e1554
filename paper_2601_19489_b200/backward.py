"""Per-Gaussian raster backward on the B200 (reference: tilesplat/backward.py).

`backward_per_gaussian` launches K4 (csrc/backward.cu).  Grad2D keeps the
reference's fields (backward.py:36-50) as views into one packed (M, 10)
buffer {d_mx, d_my, d_a, d_b, d_c, d_opacity, d_r, d_g, d_b, d_depth} that
K4 merges into with one atomic per (splat, tile, field).  `merges` follows
the reference's count: every (splat, tile) pair of every tile whose upstream
gradient is not all zero (backward.py:214-222).
"""

from __future__ import annotations

import os

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


# K4 schedule.  "regions" (default for the training step): the region-culled
# K4 (tsr_render_bwd_regions, csrc/backward_regions.cu) fed by K3's region
# lists; the public backward_per_gaussian, whose buffers carry the
# reference's checkpoints but no region lists, then runs the per-tile form.
# "tiles": one CTA per tile, its 4 warps taking the
# tile's supergroups (tsr_render_bwd).  "units": the (tile, supergroup) work
# units of the frame drained by the warps of a persistent grid
# (tsr_render_bwd_ws) -- heavy tiles spread over the GPU and no warp idles at
# a tile's end (warp slots busy 75 % -> ~94 %), but at C2 it measured 4 %
# slower: K4 is FP32-pipe bound (math-pipe throttle is the top stall and
# grows with the extra warps) and each unit re-gathers its pixel records
# (DESIGN.md §8).  TSR_K4=units selects it.
K4_FORM = os.environ.get("TSR_K4", "regions")
# pair capacity from which the training step takes the region-culled K4
REGIONS_MIN_PAIRS = int(os.environ.get("TSR_K4_REGIONS_MIN_PAIRS", 1_000_000))


def backward_regions_raw(rec, values, offsets, width: int, height: int, targets, ckpt_base,
                         regions, grad_color, grad_depth, grad_final_T, out: torch.Tensor,
                         merges: torch.Tensor) -> None:
    """Region-culled K4 (backward.py:137-223) over K3's region lists and
    work units (render_regions_raw); merges into `out` (zeroed by the caller)."""
    lib = _lib.load()
    _lib.check(lib.tsr_render_bwd_regions(
        rec.data_ptr(), _lib.ptr(values), offsets.data_ptr(), width, height,
        targets.color.data_ptr(), targets.depth.data_ptr(), targets.final_T.data_ptr(),
        targets.n_considered.data_ptr(), targets.ckpt.data_ptr(), ckpt_base.data_ptr(),
        regions.list.data_ptr(), regions.seg.data_ptr(), regions.units.data_ptr(),
        regions.ctl.data_ptr(), grad_color.data_ptr(), _lib.ptr(grad_depth),
        _lib.ptr(grad_final_T), out.data_ptr(), merges.data_ptr(), regions.height,
        _lib.stream_handle()), "tsr_render_bwd_regions")


class BackwardWorkspace:
    """Device scratch of the work-unit K4 (unit plan + queue), sized for a
    pair bound; reused across calls of the same shape."""

    def __init__(self):
        self.buf = None
        self.key = None

    def get(self, width: int, height: int, p_bound: int) -> torch.Tensor:
        if self.buf is None or self.key[0] != (width, height) or self.key[1] < p_bound:
            n = int(_lib.load().tsr_render_bwd_workspace(width, height, p_bound))
            self.buf = torch.empty(n, dtype=torch.uint8, device=_device())
            self.key = ((width, height), p_bound)
        return self.buf


def backward_per_gaussian_raw(buffers: RenderBuffers, batch: SplatBatch, tiles: TileIndex,
                              grad_color, grad_depth=None, grad_final_T=None,
                              out: torch.Tensor | None = None,
                              merges: torch.Tensor | None = None,
                              workspace: BackwardWorkspace | None = None,
                              p_bound: int | None = None) -> tuple:
    """Launch K4 without host synchronisation; returns (packed grads, merges).
    p_bound (>= the pair count; a capacity is fine) sizes the work-unit
    plan; default tiles.n_pairs."""
    lib = _lib.load()
    dev = _device()
    if out is None:
        out = torch.zeros((len(batch), _lib.GRAD2D_FLOATS), dtype=torch.float32, device=dev)
    if merges is None:
        merges = torch.zeros(1, dtype=torch.int64, device=dev)
    gc = as_device_f32(grad_color)
    gd = as_device_f32(grad_depth) if grad_depth is not None else None
    gt = as_device_f32(grad_final_T) if grad_final_T is not None else None
    common = (batch.rec.data_ptr(), _lib.ptr(tiles.values) if tiles.n_pairs else None,
              tiles.offsets.data_ptr(), batch.width, batch.height, buffers.color.data_ptr(),
              buffers.depth.data_ptr(), buffers.final_T.data_ptr(),
              buffers.n_considered.data_ptr(), _lib.ptr(buffers.ckpt),
              _lib.ptr(buffers.ckpt_base), gc.data_ptr(), _lib.ptr(gd), _lib.ptr(gt),
              out.data_ptr(), merges.data_ptr())
    if K4_FORM in ("tiles", "regions"):
        _lib.check(lib.tsr_render_bwd(*common, _lib.stream_handle()), "tsr_render_bwd")
        return out, merges
    p_bound = tiles.n_pairs if p_bound is None else p_bound
    ws = (workspace or BackwardWorkspace()).get(batch.width, batch.height, p_bound)
    _lib.check(lib.tsr_render_bwd_ws(*common, int(p_bound), ws.data_ptr(), ws.numel(),
                                     _lib.stream_handle()), "tsr_render_bwd_ws")
    return out, merges


def backward_det_raw(buffers: RenderBuffers, batch: SplatBatch, tiles: TileIndex, grad_color,
                     grad_depth, grad_final_T, out: torch.Tensor, merges: torch.Tensor,
                     slots: torch.Tensor, processed: torch.Tensor, m_dev=None,
                     workspace: BackwardWorkspace | None = None,
                     p_bound: int | None = None) -> None:
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
    common = (batch.rec.data_ptr(), _lib.ptr(tiles.values) if tiles.n_pairs else None,
              tiles.offsets.data_ptr(), batch.width, batch.height, buffers.color.data_ptr(),
              buffers.depth.data_ptr(), buffers.final_T.data_ptr(),
              buffers.n_considered.data_ptr(), _lib.ptr(buffers.ckpt),
              _lib.ptr(buffers.ckpt_base), gc.data_ptr(), _lib.ptr(gd), _lib.ptr(gt),
              merges.data_ptr(), slots.data_ptr(), processed.data_ptr(), inv_perm.data_ptr(),
              rank_row.data_ptr(), rank_count.data_ptr(), rank_off.data_ptr(),
              tiles.keys.data_ptr(), out.shape[0], _lib.ptr(m_dev), out.data_ptr())
    if K4_FORM in ("tiles", "regions"):
        _lib.check(lib.tsr_render_bwd_det(*common, _lib.stream_handle()), "tsr_render_bwd_det")
        return
    p_bound = tiles.n_pairs if p_bound is None else p_bound
    ws = (workspace or BackwardWorkspace()).get(batch.width, batch.height, p_bound)
    _lib.check(lib.tsr_render_bwd_ws_det(*common, int(p_bound), ws.data_ptr(), ws.numel(),
                                         _lib.stream_handle()), "tsr_render_bwd_ws_det")


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
