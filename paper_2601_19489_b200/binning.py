"""Tile binning on the B200 (reference: tilesplat/binning.py).

Both strategies produce the reference's bit-exact TileIndex:
  * bin_sequential      -- exact FP64 column walk (binning.py:166-222)
  * bin_load_balanced   -- warp-per-splat FP64 min-q group test, candidates
                           dealt round-robin to 32 lanes (binning.py:225-286)
then the on-device stable LSD radix sort on tile<<32 | f32 depth bits and the
per-tile ranges (binning.py:137-158).

Device layout: keys (P,) int64, values (P,) int32 batch rows, offsets (T+1,)
int64.  `ckpt_base` (T+1,) int64 = offsets >> 5: where each tile's
floor(n_tile/32) forward checkpoint records start (forward.py:139-145).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .projection import SplatBatch
from .scene import TILE, _device


@dataclass
class SnugBox:
    x_min: float
    x_max: float
    y_min: float
    y_max: float
    tile_rect: tuple


class TileIndex:
    """Depth-sorted (tile, splat) pairs with per-tile ranges (binning.py:37-71)."""

    def __init__(self, keys, values, offsets, tiles_x, tiles_y, ckpt_base=None, det=None):
        self.keys = keys
        self.values = values
        self.offsets = offsets
        self.tiles_x = int(tiles_x)
        self.tiles_y = int(tiles_y)
        self.ckpt_base = ckpt_base
        # (inv_perm, rank_row, rank_count, rank_off) for the deterministic merge
        self.det = det

    @property
    def n_pairs(self) -> int:
        return int(self.keys.shape[0])

    @property
    def n_tiles(self) -> int:
        return self.tiles_x * self.tiles_y

    def tile_range(self, tile_id: int):
        return int(self.offsets[tile_id]), int(self.offsets[tile_id + 1])

    def depths(self) -> torch.Tensor:
        return (self.keys & 0xFFFFFFFF).to(torch.int32).view(torch.float32)

    def tile_ids(self) -> torch.Tensor:
        return self.keys >> 32

    def checksum(self) -> str:
        """sha256(keys as u64 || values as i64)[:16] (binning.py:67-71)."""
        h = hashlib.sha256()
        h.update(self.keys.cpu().numpy().astype(np.uint64).tobytes())
        h.update(self.values.cpu().numpy().astype(np.int64).tobytes())
        return h.hexdigest()[:16]


def _tiles(batch: SplatBatch):
    return -(-batch.width // TILE), -(-batch.height // TILE)


def compute_snugboxes(batch: SplatBatch) -> SplatBatch:
    """Fill FP64 extents and inclusive tile rects in place (binning.py:87-104)."""
    lib = _lib.load()
    m = len(batch)
    dev = _device()
    batch.x_min = torch.empty(m, dtype=torch.float64, device=dev)
    batch.x_max = torch.empty(m, dtype=torch.float64, device=dev)
    batch.y_min = torch.empty(m, dtype=torch.float64, device=dev)
    batch.y_max = torch.empty(m, dtype=torch.float64, device=dev)
    batch.tile_rect = torch.empty((m, 4), dtype=torch.int32, device=dev)
    _lib.check(lib.tsr_snugboxes(
        batch.rec.data_ptr(), m, batch.width, batch.height, batch.x_min.data_ptr(),
        batch.x_max.data_ptr(), batch.y_min.data_ptr(), batch.y_max.data_ptr(),
        batch.tile_rect.data_ptr(), _lib.stream_handle()), "tsr_snugboxes")
    return batch


def snugbox(conic, t, mean, image_dims) -> SnugBox:
    """Single-splat SnugBox (binning.py:107-122), evaluated by the same kernel."""
    a, b, c = (float(v) for v in conic)
    if not (a > 0 and c > 0 and a * c - b * b > 0):
        raise ValueError("conic is not positive definite")
    if t < 0:
        raise ValueError("level t must be >= 0")
    width, height = image_dims
    batch = SplatBatch([mean], [conic], [t], [1.0], [1.0], [0], width, height)
    compute_snugboxes(batch)
    r = batch.tile_rect[0].tolist()
    return SnugBox(float(batch.x_min[0]), float(batch.x_max[0]), float(batch.y_min[0]),
                   float(batch.y_max[0]), tuple(int(v) for v in r))


def _ensure_counts(batch: SplatBatch, strategy: int) -> None:
    """Per-row pair counts / depth bits / spans; reuses K1's fused count when
    it was made with the same strategy."""
    if batch.counts is not None and batch.strategy == strategy:
        return
    lib = _lib.load()
    m = len(batch)
    dev = _device()
    batch.counts = torch.empty(max(m, 1), dtype=torch.int32, device=dev)[:m]
    batch.depth_bits = torch.empty(max(m, 1), dtype=torch.int32, device=dev)[:m]
    batch.spans = torch.empty((max(m, 1), 4), dtype=torch.int32, device=dev)[:m]
    batch.totals = torch.zeros(2, dtype=torch.int64, device=dev)
    _lib.check(lib.tsr_count_pairs(batch.rec.data_ptr(), m, batch.width, batch.height, strategy,
                                   batch.counts.data_ptr(), batch.depth_bits.data_ptr(),
                                   batch.spans.data_ptr(), batch.totals.data_ptr(),
                                   _lib.stream_handle()), "tsr_count_pairs")
    batch.n_pairs = int(batch.totals[1].item())
    batch.strategy = strategy


class IndexBuffers:
    """Capacity buffers for K2 (reused across steps by the trainer)."""

    def __init__(self, m_cap: int, p_cap: int, n_tiles: int, det: bool = False):
        dev = _device()
        lib = _lib.load()
        self.m_cap, self.p_cap, self.n_tiles = m_cap, p_cap, n_tiles
        self.det = None
        if det:  # K2's outputs for the deterministic merge
            u32 = torch.int32
            self.det = (torch.empty(max(p_cap, 1), dtype=u32, device=dev),
                        torch.empty(max(m_cap, 1), dtype=u32, device=dev),
                        torch.empty(max(m_cap, 1), dtype=u32, device=dev),
                        torch.empty(max(m_cap, 1), dtype=u32, device=dev))
        self.keys = torch.empty(max(p_cap, 1), dtype=torch.int64, device=dev)
        self.values = torch.empty(max(p_cap, 1), dtype=torch.int32, device=dev)
        self.offsets = torch.empty(n_tiles + 1, dtype=torch.int64, device=dev)
        self.ckpt_base = torch.empty(n_tiles + 1, dtype=torch.int64, device=dev)
        self.overflow = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ws_bytes = int(lib.tsr_index_workspace(m_cap, p_cap))
        self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)

    def fits(self, m: int, p: int, n_tiles: int) -> bool:
        return m <= self.m_cap and p <= self.p_cap and n_tiles == self.n_tiles


def build_index_raw(batch: SplatBatch, strategy: int, bufs: IndexBuffers) -> None:
    """Launch K2 into capacity buffers; sizes come from batch.totals on the device."""
    lib = _lib.load()
    args = (batch.rec.data_ptr(), batch.depth_bits.data_ptr(), batch.spans.data_ptr(),
            batch.counts.data_ptr(), batch.totals.data_ptr(), bufs.m_cap, bufs.p_cap,
            batch.width, batch.height, strategy, bufs.keys.data_ptr(), bufs.values.data_ptr(),
            bufs.offsets.data_ptr(), bufs.ckpt_base.data_ptr(), bufs.overflow.data_ptr(),
            bufs.workspace.data_ptr(), bufs.ws_bytes)
    if bufs.det is not None:
        _lib.check(lib.tsr_build_index_det(*args, *(t.data_ptr() for t in bufs.det),
                                           _lib.stream_handle()), "tsr_build_index_det")
    else:
        _lib.check(lib.tsr_build_index(*args, _lib.stream_handle()), "tsr_build_index")


def build_index(batch: SplatBatch, strategy: int, bufs: IndexBuffers | None = None) -> TileIndex:
    """K2 with exact sizes (one host read of P when not already known)."""
    _ensure_counts(batch, strategy)
    tiles_x, tiles_y = _tiles(batch)
    m, p = len(batch), int(batch.n_pairs)
    if bufs is None or not bufs.fits(m, p, tiles_x * tiles_y):
        bufs = IndexBuffers(m, p, tiles_x * tiles_y, det=True)
    build_index_raw(batch, strategy, bufs)
    return TileIndex(bufs.keys[:p], bufs.values[:p], bufs.offsets, tiles_x, tiles_y,
                     bufs.ckpt_base, bufs.det)


def bin_sequential(batch: SplatBatch) -> TileIndex:
    """Column-walk binning (binning.py:166-222)."""
    return build_index(batch, 0)


def bin_load_balanced(batch: SplatBatch, group_size: int = 32) -> TileIndex:
    """Group-testing binning (binning.py:262-286); identical output."""
    if group_size != 32:
        raise ValueError("the sm_100a kernel deals candidates to one 32-lane warp")
    return build_index(batch, 1)


def bin_aabb(batch: SplatBatch) -> TileIndex:
    """Radius-rectangle baseline (binning.py:301-325): every tile of the square
    of half-side sqrt(t / lambda_min) around the mean, no intersection test."""
    return build_index(batch, 2)


def lane_test_counts(batch: SplatBatch, splat_row: int, group_size: int = 32):
    """Candidates tested per lane for one splat (binning.py:289-298)."""
    if batch.tile_rect is None:
        compute_snugboxes(batch)
    r = [int(v) for v in batch.tile_rect[splat_row].tolist()]
    n = max(0, r[1] - r[0] + 1) * max(0, r[3] - r[2] + 1)
    counts = np.zeros(group_size, dtype=np.int64)
    full, rem = divmod(n, group_size)
    counts[:] = full
    counts[:rem] += 1
    return counts
