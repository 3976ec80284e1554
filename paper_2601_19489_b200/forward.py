"""Tile rasterizer forward on the B200 (reference: tilesplat/forward.py).

`render` launches K3 (csrc/render.cu).  Checkpoints are one flat FP32 buffer:
record r of tile t is the (T, Cr, Cg, Cb, D) state after list position
32(r+1)-1, stored at ckpt[ckpt_base[t] + r] as a (5, 256) plane (forward.py:
139-140), written for every pixel that consumed that position.  The
reference's padding records for already-terminated pixels are never written
because the backward never reads them (it enters group g of a pixel only if
n_considered > 32 g); `checkpoints_dict()` materialises the reference's
{tile: (G, 5, th, tw)} view for inspection.
"""

from __future__ import annotations

import os

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .binning import TileIndex
from .projection import MIN_OPACITY, SplatBatch
from .scene import TILE, _device

ALPHA_CAP = 0.99
MIN_ALPHA = MIN_OPACITY
T_TERMINATE = 1e-4
CHECKPOINT_INTERVAL = 32


@dataclass
class RenderBuffers:
    color: torch.Tensor        # (H, W, 3), background composited in
    depth: torch.Tensor        # (H, W)
    final_T: torch.Tensor      # (H, W)
    n_contrib: torch.Tensor    # (H, W) int32
    n_considered: torch.Tensor # (H, W) int32
    background: np.ndarray
    ckpt: torch.Tensor | None = None       # flat checkpoint records
    ckpt_base: torch.Tensor | None = None  # (T+1,) record base per tile
    tiles_x: int = 0
    tiles_y: int = 0
    _ckpt_dict: dict | None = field(default=None, repr=False)

    @property
    def has_checkpoints(self) -> bool:
        return self.ckpt is not None

    def normalized_depth(self) -> torch.Tensor:
        """Depth / (1 - final_T) where anything blended (forward.py:44-50)."""
        mask = self.n_contrib > 0
        denom = torch.where(mask, 1.0 - self.final_T, torch.ones_like(self.final_T))
        return torch.where(mask, self.depth / denom, torch.zeros_like(self.depth))

    def checkpoints_dict(self, tiles: TileIndex) -> dict:
        """{tile: (G, 5, th, tw)} like the reference (entries of pixels that did
        not reach a record's position are unspecified)."""
        if self.ckpt is None:
            return {}
        out = {}
        base = self.ckpt_base.cpu().numpy()
        offs = tiles.offsets.cpu().numpy()
        H, W = self.color.shape[:2]
        flat = self.ckpt.view(-1, 5, TILE, TILE)
        for t in range(tiles.n_tiles):
            g = int(offs[t + 1] - offs[t]) // CHECKPOINT_INTERVAL
            if g == 0:
                continue
            ty, tx = divmod(t, tiles.tiles_x)
            th = min(TILE, H - ty * TILE)
            tw = min(TILE, W - tx * TILE)
            out[t] = flat[int(base[t]): int(base[t]) + g, :, :th, :tw]
        return out

    @property
    def checkpoints(self) -> dict:
        raise AttributeError("use checkpoints_dict(tiles): device checkpoints are a flat buffer")


def tile_window(tile_id: int, tiles_x: int, width: int, height: int):
    """Pixel bounds of one tile (forward.py:61-68)."""
    ty, tx = divmod(tile_id, tiles_x)
    x0, y0 = tx * TILE, ty * TILE
    return x0, y0, min(x0 + TILE, width), min(y0 + TILE, height)


def _ensure_colors(batch: SplatBatch, colors) -> None:
    """The raster record carries RGB at rec[:, 8:11]; copy caller colours in
    unless they already are that view."""
    if isinstance(colors, torch.Tensor) and colors.is_cuda:
        rc = batch.rec[:, 8:11]
        if colors.data_ptr() == rc.data_ptr() and colors.stride() == rc.stride():
            return
    if len(batch) == 0:
        return
    batch.rec[:, 8:11] = torch.as_tensor(np.asarray(colors, dtype=np.float32)
                                         if not isinstance(colors, torch.Tensor) else colors,
                                         device=batch.rec.device).reshape(-1, 3).float()


class RenderTargets:
    """Preallocated forward outputs (reused across steps by the trainer)."""

    def __init__(self, height: int, width: int, ckpt_records: int | None):
        dev = _device()
        self.color = torch.empty((height, width, 3), dtype=torch.float32, device=dev)
        self.depth = torch.empty((height, width), dtype=torch.float32, device=dev)
        self.final_T = torch.empty((height, width), dtype=torch.float32, device=dev)
        self.n_contrib = torch.empty((height, width), dtype=torch.int32, device=dev)
        self.n_considered = torch.empty((height, width), dtype=torch.int32, device=dev)
        self.ckpt = None
        if ckpt_records is not None:
            self.ckpt = torch.empty(max(ckpt_records, 1) * 5 * TILE * TILE, dtype=torch.float32,
                                    device=dev)


@dataclass
class Contributions:
    """Strong contributions (w = T alpha >= 1/255) of a scoring render
    (forward.py:53-58): parallel int64 device arrays.  The multiset equals
    the reference's; the order is (tile, warp block, list position, lane)
    instead of (tile, list position, row-major pixel)."""
    pixel_idx: torch.Tensor
    splat_rows: torch.Tensor


def render_score_raw(rec, values, offsets, width: int, height: int, background, out: RenderTargets,
                     mode: int, *, mask=None, weight: float = 0.0, row_score=None,
                     warp_counts=None, warp_base=None, out_pixel=None, out_row=None) -> None:
    """Launch K3 in scoring mode 1 (count), 2 (write) or 3 (masked row score)."""
    lib = _lib.load()
    bg = np.asarray(background, dtype=np.float64).reshape(3)
    bg_host = (_lib.c_f32 * 3)(*[float(v) for v in bg])
    _lib.check(lib.tsr_render_score(
        rec.data_ptr(), _lib.ptr(values), offsets.data_ptr(), width, height, bg_host, mode,
        _lib.ptr(mask), float(weight), _lib.ptr(row_score), _lib.ptr(warp_counts),
        _lib.ptr(warp_base), _lib.ptr(out_pixel), _lib.ptr(out_row), out.color.data_ptr(),
        out.depth.data_ptr(), out.final_T.data_ptr(), out.n_contrib.data_ptr(),
        out.n_considered.data_ptr(), _lib.stream_handle()), "tsr_render_score")


def render_raw(rec, values, offsets, ckpt_base, width: int, height: int, background,
               out: RenderTargets, ckpt_stride: int = 1, tile_order=None) -> None:
    """Launch K3 into preallocated targets (no host synchronisation).
    ckpt_stride 2 writes only the checkpoint records K4 reads (training step);
    tile_order (device int32, tsr_tile_order) launches heavy tiles first."""
    lib = _lib.load()
    bg = np.asarray(background, dtype=np.float64).reshape(3)
    bg_host = (_lib.c_f32 * 3)(*[float(v) for v in bg])
    _lib.check(lib.tsr_render_fwd_ordered(
        rec.data_ptr(), _lib.ptr(values), offsets.data_ptr(), width, height, bg_host,
        out.color.data_ptr(), out.depth.data_ptr(), out.final_T.data_ptr(),
        out.n_contrib.data_ptr(), out.n_considered.data_ptr(), _lib.ptr(out.ckpt),
        _lib.ptr(ckpt_base) if out.ckpt is not None else None, int(ckpt_stride),
        _lib.ptr(tile_order), _lib.stream_handle()), "tsr_render_fwd_ordered")


# 8x8 regions by default (4 per tile; K4r: 8-lane pipelines of 8 pixels per
# lane, TSR_K4R_PX=4: 16 lanes of 4); 8x4 with TSR_K4R_REGION=4
REGION_HEIGHT = int(os.environ.get("TSR_K4R_REGION", 8))


class RegionLists:
    """Per-(tile, region) list positions K3 writes for the region-culled
    K4 (tsr_render_fwd_regions): one list slot per region and pair, the
    segment-boundary offsets and the backward's work-unit queue; sized for a
    pair bound, reused across steps."""

    def __init__(self, width: int, height: int, p_bound: int, region_height: int | None = None):
        lib = _lib.load()
        # 8x4 regions (8 per tile, 8-lane backward pipelines) or 8x8 (4 per tile, 16 lanes)
        self.height = int(region_height or REGION_HEIGHT)
        dev = _device()
        self.list = torch.empty(int(lib.tsr_region_list_entries(width, height, p_bound)),
                                dtype=torch.int32, device=dev)
        self.seg = torch.empty(int(lib.tsr_region_seg_entries(width, height, p_bound)),
                               dtype=torch.int32, device=dev)
        self.units = torch.empty(int(lib.tsr_region_unit_entries(width, height, p_bound)),
                                 dtype=torch.int32, device=dev)
        # per-bucket unit counts + the backward's grab counter (zeroed by K3's launch)
        self.ctl = torch.zeros(int(lib.tsr_region_ctl_entries()), dtype=torch.int32, device=dev)
        self.shape = (width, height, p_bound)


def render_regions_raw(rec, values, offsets, ckpt_base, width: int, height: int, background,
                       out: RenderTargets, regions: RegionLists, tile_order=None) -> None:
    """K3 for the region-culled backward: checkpoint records at segment
    starts only plus the region lists (no host synchronisation)."""
    lib = _lib.load()
    bg = np.asarray(background, dtype=np.float64).reshape(3)
    bg_host = (_lib.c_f32 * 3)(*[float(v) for v in bg])
    _lib.check(lib.tsr_render_fwd_regions(
        rec.data_ptr(), _lib.ptr(values), offsets.data_ptr(), width, height, bg_host,
        out.color.data_ptr(), out.depth.data_ptr(), out.final_T.data_ptr(),
        out.n_contrib.data_ptr(), out.n_considered.data_ptr(), out.ckpt.data_ptr(),
        ckpt_base.data_ptr(), regions.list.data_ptr(), regions.seg.data_ptr(),
        regions.units.data_ptr(), regions.ctl.data_ptr(), regions.height, _lib.ptr(tile_order),
        _lib.stream_handle()), "tsr_render_fwd_regions")


# per-tile kernel launch order in the training step: "heavy" (heavy tiles
# first, tsr_tile_order) or "raster"
TILE_ORDER = os.environ.get("TSR_TILE_ORDER", "heavy")


def render(batch: SplatBatch, tiles: TileIndex, colors, background, *,
           record_checkpoints: bool = True, scoring: bool = False):
    """K3 forward (forward.py:87-161)."""
    _ensure_colors(batch, colors)
    H, W = batch.height, batch.width
    bg = np.asarray(background, dtype=np.float64).reshape(3)
    # sum_t floor(n_t / 32) <= P / 32 records of 5 x 256 floats
    out = RenderTargets(H, W, tiles.n_pairs // CHECKPOINT_INTERVAL + 1
                        if record_checkpoints else None)
    render_raw(batch.rec, tiles.values if tiles.n_pairs else None, tiles.offsets,
               tiles.ckpt_base, W, H, bg, out)
    color, depth, final_T, n_contrib, n_cons, ckpt = (out.color, out.depth, out.final_T,
                                                      out.n_contrib, out.n_considered, out.ckpt)
    bufs = RenderBuffers(color, depth, final_T, n_contrib, n_cons, bg, ckpt,
                         tiles.ckpt_base if ckpt is not None else None,
                         tiles.tiles_x, tiles.tiles_y)
    if not scoring:
        return bufs
    return bufs, contributions(batch, tiles, bg)


def contributions(batch: SplatBatch, tiles: TileIndex, background) -> Contributions:
    """Scoring render (forward.py:132-137): count the strong contributions per
    (tile, warp), scan, then write them (two K3 launches in scoring mode)."""
    H, W = batch.height, batch.width
    dev = _device()
    scratch = RenderTargets(H, W, None)
    n_slots = tiles.n_tiles * 4
    counts = torch.zeros(n_slots, dtype=torch.int64, device=dev)
    values = tiles.values if tiles.n_pairs else None
    render_score_raw(batch.rec, values, tiles.offsets, W, H, background, scratch, 1,
                     warp_counts=counts)
    base = torch.cumsum(counts, 0) - counts
    total = int(counts.sum().item())
    pix = torch.empty(max(total, 1), dtype=torch.int64, device=dev)[:total]
    rows = torch.empty(max(total, 1), dtype=torch.int64, device=dev)[:total]
    if total:
        render_score_raw(batch.rec, values, tiles.offsets, W, H, background, scratch, 2,
                         warp_base=base, out_pixel=pix, out_row=rows)
    return Contributions(pix, rows)
