"""Training-step glue on the B200 (reference: tilesplat/trainer.py:181-257).

`render_view`, `view_loss_and_grads` and `_full_grads` keep the reference's
names and return types.  `TrainStep` is the hot path the benchmark times: one
view through K1 (project+count) -> K2 (duplicate, sort, ranges) -> K3 render
-> loss -> K4 backward -> K4b+K5 fused projection-VJP + Adam, with a single
host read of the pair count (P sizes the key buffers).
"""

from __future__ import annotations

import json
import os

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, losses
from .backward import Grad2D, backward_per_gaussian, backward_per_gaussian_raw
from .binning import TileIndex, build_index
from .forward import RenderBuffers, render
from .optim import Adam, position_lr
from .pose import PoseDelta
from .projection import (ProjectionScratch, SplatBatch, _pose_grad_from_sums, batch_from_scratch,
                         camera_struct,
                         gaussians_struct, project, project_raw, project_vjp)
from .scene import Camera, GaussianSet, _device, as_device_f32

_PROFILE_DEFAULTS = {
    "round1": {"max_iters": 6000, "pose_opt": True, "depth_supervision": False},
    "round2": {"max_iters": 15000, "pose_opt": False, "depth_supervision": True},
}


@dataclass
class TrainConfig:
    """The reference TrainConfig (trainer.py:42-113): same names, defaults
    and validation."""
    round_profile: str = "round2"
    max_iters: int | None = None
    budget_seconds: float = 60.0
    pose_opt: bool | None = None
    depth_supervision: bool | None = None

    lambda_: float = 0.2
    depth_weight0: float = 0.1

    densify: bool = True
    densify_interval: int = 300
    densify_start: int = 500
    densify_end: int | None = None  # defaults to 0.8 * max_iters
    consistency_views: int = 10  # K
    error_tau: float = 0.5
    theta_plus: float = 16.0
    theta_minus: float = 0.9
    scale_split_threshold_frac: float = 0.01
    min_splats: int = 16

    pose_bake_interval: int = 300

    sh_degree: int = 0
    background: tuple = (0.0, 0.0, 0.0)
    near: float = 0.01
    seed: int = 0
    eval_interval: int = 100
    holdout_views: tuple = ()
    deterministic: bool = True
    threads: int = 1
    binning_strategy: str = "sequential"  # sequential | load_balanced
    backward_path: str = "per_gaussian"
    init_opacity: float = 0.1
    lrs: dict = field(default_factory=dict)

    colmap_dir: str | None = None
    images_dir: str | None = None
    depth_dir: str | None = None
    output_dir: str | None = None
    depth_samples_per_view: int = 0

    def __post_init__(self):
        if self.round_profile not in _PROFILE_DEFAULTS:
            raise ValueError(f"unknown round_profile {self.round_profile!r}")
        prof = _PROFILE_DEFAULTS[self.round_profile]
        if self.max_iters is None:
            self.max_iters = prof["max_iters"]
        if self.pose_opt is None:
            self.pose_opt = prof["pose_opt"]
        if self.depth_supervision is None:
            self.depth_supervision = prof["depth_supervision"]
        if self.densify_end is None:
            self.densify_end = int(0.8 * self.max_iters)
        if self.budget_seconds <= 0:
            raise ValueError("budget_seconds must be > 0")
        if self.binning_strategy not in ("sequential", "load_balanced"):
            raise ValueError(f"unknown binning_strategy {self.binning_strategy!r}")
        if self.backward_path != "per_gaussian":
            raise ValueError("only the per-Gaussian backward is built for the GPU "
                             "(backward_per_pixel is the CPU oracle)")

    @classmethod
    def from_json(cls, path) -> "TrainConfig":
        import json
        with open(path) as fh:
            data = json.load(fh)
        unknown = set(data) - set(cls.__dataclass_fields__)
        if unknown:
            raise ValueError(f"unknown config keys: {sorted(unknown)}")
        return cls(**data)

    def to_json(self, path) -> None:
        import json
        from dataclasses import asdict
        with open(path, "w") as fh:
            json.dump(asdict(self), fh, indent=2, default=list)

    @property
    def strategy_id(self) -> int:
        return 1 if self.binning_strategy == "load_balanced" else 0


@dataclass
class ViewRender:
    batch: SplatBatch
    tiles: TileIndex
    colors: torch.Tensor
    dirs: object
    buffers: RenderBuffers
    contributions: object = None


def render_view(gset: GaussianSet, camera: Camera, cfg: TrainConfig,
                delta: PoseDelta | None = None, *, checkpoints: bool = True,
                scoring: bool = False) -> ViewRender:
    """project -> bin -> colours -> render (trainer.py:181-192)."""
    batch = project(gset, camera, near=cfg.near, delta=delta, strategy=cfg.strategy_id)
    tiles = build_index(batch, cfg.strategy_id)
    colors = batch.colors
    out = render(batch, tiles, colors, cfg.background, record_checkpoints=checkpoints,
                 scoring=scoring)
    if scoring:
        bufs, contribs = out
        return ViewRender(batch, tiles, colors, None, bufs, contribs)
    return ViewRender(batch, tiles, colors, None, out)


def view_loss_and_grads(camera: Camera, cfg: TrainConfig, vr: ViewRender,
                        depth_weight: float):
    """Photometric (+ disparity) loss and the raster backward (trainer.py:195-228)."""
    bufs = vr.buffers
    report, grad_color = losses.photometric(bufs.color, camera.gt_image, cfg.lambda_)
    grad_depth = grad_final_T = None
    depth_loss = 0.0
    if depth_weight > 0.0 and camera.depth_prior is not None:
        # fused disparity loss + chain through d_norm = D / (1 - T_f)
        dl, grad_depth, grad_final_T, _ = losses.depth_chain_device(
            bufs.depth, bufs.final_T, bufs.n_contrib, camera.depth_prior, camera.depth_valid,
            depth_weight)
        depth_loss = float(dl.item())
    g2 = backward_per_gaussian(bufs, vr.batch, vr.tiles, vr.colors, grad_color, grad_depth,
                               grad_final_T)
    report = losses.LossReport(l1=report.l1, ssim=report.ssim, photometric=report.photometric,
                               depth_loss=depth_loss, total=report.photometric + depth_loss,
                               lambda_=cfg.lambda_, depth_weight=depth_weight)
    return report, g2


def _full_grads(gset: GaussianSet, camera: Camera, cfg: TrainConfig, delta, vr: ViewRender,
                g2: Grad2D) -> dict:
    """project_vjp + colour chain, keyed like the optimizer groups (trainer.py:231-257)."""
    gcol = torch.empty_like(gset.colors)
    g3, gpose = project_vjp(gset, camera, vr.batch, g2, near=cfg.near, delta=delta,
                            grad_colors=gcol)
    return {"positions": g3.positions, "log_scales": g3.log_scales,
            "rotations": g3.rotations, "opacity_logits": g3.opacity_logits,
            "colors": gcol, "pose_rot": gpose.rot_vec, "pose_trans": gpose.trans}


# TSR_FUSED_ADAM=1: the SH-0 step runs the projection VJP + Adam fused into
# K4's tail (tsr_render_bwd_adam: per-row merge counters, the CTA completing a
# row updates it).  Measured slower at C2 (K4 575 -> 1177 us, + 55 us for the
# rows without pairs, against 86 us for the separate K4b+K5 kernel): each
# tile CTA's counting atomics and its HBM-latency-bound updates hold the SM
# slot the FP32-bound backward needs, so it is opt-in.
FUSED_ADAM = os.environ.get("TSR_FUSED_ADAM", "0") == "1"


class TrainStep:
    """One-view training step on the device (fwd + loss + bwd + Adam).

    Hot path for BASELINE.json's metric; the reference's per-step sequence is
    trainer.py:329-345.  Positions use the decaying lr (position_lr) exactly as
    the reference loop does; pose optimisation is off (round2 profile).

    The step never synchronises with the host: every size (M rows, P pairs)
    stays on the device and all buffers are capacity-allocated.  The pair
    capacity is sized with headroom from the first step's P, or up front
    from the largest P over a camera set (`reserve`).  K2 raises a sticky
    overflow flag; the fused VJP + Adam kernel reads it and skips the update
    of an overflowed step (its tile lists were truncated), counting the
    skipped steps on the device.  The host polls the flag without blocking
    (a pinned copy + event from an earlier step); on overflow it grows the
    capacity, rolls the Adam step counters back and redoes the skipped steps
    from its history, so training proceeds exactly as with enough capacity.
    Capacity also grows pre-emptively at 80 % occupancy."""

    HISTORY = 64  # steps kept for redo (bounds how far the host may run ahead)

    def __init__(self, gset: GaussianSet, cfg: TrainConfig, extent: float = 4.0,
                 optimizer: Adam | None = None, p_headroom: float = 1.5, graphs: bool = False,
                 deterministic: bool | None = None):
        self.gset = gset
        self.cfg = cfg
        # deterministic merge in K4: bitwise run-to-run reproducible (opt-in;
        # the default atomic merge agrees within FP32 rounding).  The
        # reference's cfg.deterministic concerns its CPU worker pool.
        self.deterministic = bool(deterministic)
        self.slots = None
        self.processed = None
        # CUDA-graph replay of the whole step (after the first, eager, step
        # has sized the capacities): one graph per (camera, GT buffer, depth
        # inputs), each with its own private memory pool.  Per-step scalars
        # (Adam lr and bias corrections, the depth weight) reach the kernels
        # through pinned-memory copy nodes.
        self.graphs = graphs
        self._graph_cache = {}
        # device copy the graph reads: [lr, bc1, bc2] x 5 groups, depth weight
        self._scal_dev = torch.zeros(16, dtype=torch.float32, device=_device())
        # host staging ring: slot k is copied (stream-ordered, before the
        # replay) into _scal_dev and not rewritten until its copy completed,
        # so the host may run ahead of the device by up to kRing steps
        self._ring = [torch.zeros(16, dtype=torch.float32).pin_memory() for _ in range(8)]
        self._ring_ev = [None] * 8
        self._ring_k = 0
        self.opt = optimizer or Adam({k: v for k, v in cfg.lrs.items() if k != "positions"})
        self.pos_base_lr = cfg.lrs.get("positions", 1.6e-4 * extent)
        self.iteration = 0
        self.p_headroom = p_headroom
        n = len(gset)
        dev = _device()
        self.scratch = ProjectionScratch(n)
        self.index = None
        self.targets = None
        self.hw = None
        self.grad2d = torch.zeros((max(n, 1), _lib.GRAD2D_FLOATS), dtype=torch.float32,
                                  device=dev)
        self.skipped = torch.zeros(1, dtype=torch.int64, device=dev)
        # overflowed steps whose update the fused kernel skipped (device)
        self.gated_steps = torch.zeros(1, dtype=torch.int32, device=dev)
        # per-row merge counters of the fused K4 + update (zero between steps)
        self.row_done = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        self._updated = False
        self._history = []  # (camera, gt, depth args, iteration, loss tensors) per step
        self.redone_steps = 0
        self.merges = torch.zeros(1, dtype=torch.int64, device=dev)
        self.loss_ws = losses.PhotometricWorkspace()
        # recorded once the step's loss kernels have read the GT image (also
        # inside a captured step: an external event node), so a host-fed loop
        # may refill that GT buffer while the backward still runs
        self.gt_consumed = torch.cuda.Event(external=True)
        from .backward import BackwardWorkspace
        self.bwd_ws = BackwardWorkspace()
        self.regions = None
        self._order_buf = None
        self.tile_order = None
        self.dc_ws = losses.DepthChainWorkspace()
        self._grad2d_clean = True  # the SH-0 fused kernel re-zeroes consumed rows
        self.grad_color = None
        # step status read back without kernels: two D2H copy nodes into
        # pinned memory (overflow flag; totals = (M, P))
        self.status_ovf_host = torch.zeros(1, dtype=torch.int32).pin_memory()
        self.status_tot_host = torch.zeros(2, dtype=torch.int64).pin_memory()
        self.status_event = None
        self.lib = _lib.load()
        self.last_camera = None
        self.last = None
        self.last_losses = None

    @staticmethod
    def _mark(timer, name):
        if timer is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            timer.setdefault("_events", []).append((name, ev))

    # -------------------------------------------------------------- capacity
    def _ensure_capacity(self, camera: Camera) -> None:
        hw = (camera.height, camera.width)
        tiles = camera.tiles_x * camera.tiles_y
        if self.index is not None and self.hw == hw and self.index.n_tiles == tiles:
            return
        torch.cuda.current_stream().synchronize()      # once: size P
        p = int(self.scratch.totals[1].item())
        self._allocate(camera, int(p * self.p_headroom) + 65536)

    def _allocate(self, camera: Camera, p_cap: int) -> None:
        from .binning import IndexBuffers
        from .forward import RenderTargets
        tiles = camera.tiles_x * camera.tiles_y
        self.index = IndexBuffers(len(self.gset), p_cap, tiles, det=self.deterministic)
        self.targets = RenderTargets(camera.height, camera.width, p_cap // 32 + tiles + 1)
        self.regions = None
        if self._regions_on(p_cap):  # K3's region lists for the region-culled K4
            from .forward import RegionLists
            self.regions = RegionLists(camera.width, camera.height, p_cap)
        self.hw = (camera.height, camera.width)
        self.grad_color = torch.empty((camera.height, camera.width, 3), dtype=torch.float32,
                                      device=self.grad2d.device)
        if self.deterministic:
            self.slots = torch.empty((max(p_cap, 1), _lib.GRAD2D_FLOATS), dtype=torch.float32,
                                     device=self.grad2d.device)
            self.processed = torch.zeros(tiles, dtype=torch.int32, device=self.grad2d.device)

    def reserve(self, cameras) -> int:
        """Size the pair capacity for a camera set up front: K1 runs for
        every camera (no binning), the largest pair count is read back with
        ONE host synchronisation, and the buffers are allocated for it with
        headroom.  Returns the largest P."""
        cams = list(cameras)
        if not cams:
            raise ValueError("reserve() needs at least one camera")
        totals = []
        for cam in cams:
            project_raw(self.gset, cam, self.cfg.near, None, self.cfg.strategy_id, self.scratch)
            totals.append(self.scratch.totals[1].clone())
        p_max = int(torch.stack(totals).max().item())
        big = max(cams, key=lambda c: c.width * c.height)
        if self.index is None or int(p_max * self.p_headroom) + 65536 > self.index.p_cap:
            self._allocate(big, int(p_max * self.p_headroom) + 65536)
        return p_max

    def _poll_status(self, camera: Camera) -> None:
        """Non-blocking check of an earlier step's overflow flag and P."""
        if self.status_event is None or not self.status_event.query():
            return
        overflow, p = int(self.status_ovf_host[0]), int(self.status_tot_host[1])
        self.status_event = None
        if overflow:
            self._recover_overflow(camera)
            return
        if p > 0.8 * self.index.p_cap:
            self._allocate(camera, int(p * self.p_headroom) + 65536)
            self._graph_cache.clear()

    def _recover_overflow(self, camera: Camera) -> None:
        """Grow the pair capacity and redo the steps whose update the fused
        kernel skipped (the most recent ones: the overflow flag is sticky)."""
        torch.cuda.current_stream().synchronize()
        n_skip = int(self.gated_steps.item())
        if n_skip > len(self._history):
            raise RuntimeError(f"{n_skip} overflowed steps exceed the redo history "
                               f"({len(self._history)})")
        redo = self._history[len(self._history) - n_skip:] if n_skip else []
        # the largest P among the skipped views sizes the new capacity
        p_need = self.reserve([h[0] for h in redo] or [camera])
        self.gated_steps.zero_()
        self._graph_cache.clear()
        for name in self.opt._steps:
            if name in self.gset.params():
                self.opt._steps[name] -= n_skip
        del self._history[len(self._history) - n_skip:]
        for cam, gt, dw, dp, dv, it, outs in redo:
            self.iteration = it - 1
            self._eager_step(cam, gt, None, dw, dp, dv)
            if outs is not None:
                for old, new in zip(outs, self.last_losses):
                    if old is not None and new is not None:
                        old.copy_(new)
                self.last_losses = outs
        self.redone_steps += n_skip
        torch.cuda.current_stream().synchronize()
        if int(self.index.overflow.item()):
            raise RuntimeError(f"pair capacity still overflowed after growing to "
                               f"{self.index.p_cap} (P >= {p_need})")

    # ------------------------------------------------------------------ step
    def forward(self, camera: Camera, timer=None):
        """K1 + K2 + K3 into the capacity buffers (no host synchronisation)."""
        self._mark(timer, "start")
        project_raw(self.gset, camera, self.cfg.near, None, self.cfg.strategy_id, self.scratch)
        self._mark(timer, "preprocess")
        self._ensure_capacity(camera)
        s = self.scratch
        batch = SplatBatch(None, None, None, None, None, s.source_ids, camera.width,
                           camera.height, _rec=s.rec)
        batch.row_of_source, batch.counts, batch.depth_bits = s.row_of_source, s.counts, s.depth_bits
        batch.spans, batch.totals, batch.strategy = s.spans, s.totals, self.cfg.strategy_id
        from .binning import build_index_raw
        from .forward import render_raw
        build_index_raw(batch, self.cfg.strategy_id, self.index)
        idx, out = self.index, self.targets
        from .forward import TILE_ORDER
        self.tile_order = None
        if TILE_ORDER == "heavy":  # heavy tiles first in K3 and K4
            n_tiles = camera.tiles_x * camera.tiles_y
            if self._order_buf is None or self._order_buf.numel() != n_tiles + 1:
                self._order_buf = torch.empty(n_tiles + 1, dtype=torch.int32,
                                              device=s.rec.device)
            self.tile_order = self._order_buf
            _lib.check(self.lib.tsr_tile_order(idx.offsets.data_ptr(), n_tiles,
                                               self.tile_order.data_ptr(), _lib.stream_handle()),
                       "tsr_tile_order")
        self._mark(timer, "binning")
        if self.regions is not None:
            from .forward import render_regions_raw
            render_regions_raw(s.rec, idx.values, idx.offsets, idx.ckpt_base, camera.width,
                               camera.height, self.cfg.background, out, self.regions,
                               tile_order=self.tile_order)
        else:
            render_raw(s.rec, idx.values, idx.offsets, idx.ckpt_base, camera.width,
                       camera.height, self.cfg.background, out,
                       ckpt_stride=2,  # only the records K4 reads
                       tile_order=self.tile_order)
        self._mark(timer, "render")
        return batch

    def _regions_on(self, p_cap: int) -> bool:
        """The training step runs the region-culled K3/K4 pair (the
        deterministic merge keeps the per-tile K4 and its per-pair slots).
        Small frames keep the per-tile K4: the region K4's units (tile, row
        pair, 1024-position segment) are too few to fill the GPU there (C1:
        ~500 units for ~2,400 warp slots; measured 101 vs 61 us)."""
        from .backward import K4_FORM, REGIONS_MIN_PAIRS
        return (K4_FORM == "regions" and not self.deterministic and not self._can_fuse_update()
                and p_cap >= REGIONS_MIN_PAIRS)

    def _can_fuse_update(self) -> bool:
        from .backward import K4_FORM
        return (FUSED_ADAM and K4_FORM == "tiles" and not self.deterministic
                and self.gset.colors.shape[1] == 1)

    def loss_and_backward(self, batch, camera: Camera, gt_image, timer=None,
                          depth_weight: float = 0.0, depth_prior=None, depth_valid=None,
                          update=None):
        """Loss + K4.  update = (Adam group descriptors, device scalars or
        None): with the SH-0 per-tile K4, the projection VJP and Adam run
        fused into K4's tail (tsr_render_bwd_adam) and self._updated is set;
        otherwise the caller launches the fused K4b+K5 kernel."""
        self._updated = False
        out, idx = self.targets, self.index
        e, l1, s, grad_color = losses.photometric_device(out.color, gt_image, self.cfg.lambda_,
                                                         grad=self.grad_color,
                                                         workspace=self.loss_ws)
        self.gt_consumed.record()  # the GT image's last reader is the loss pair
        gd = gt = None
        dl = None
        # (a tensor weight comes from graph capture: no host read of it)
        if depth_prior is not None and (isinstance(depth_weight, torch.Tensor)
                                        or depth_weight > 0.0):
            dl, gd, gt, e = losses.depth_chain_device(out.depth, out.final_T, out.n_contrib,
                                                      depth_prior, depth_valid, depth_weight,
                                                      e_photo=e, workspace=self.dc_ws)
        self.last_losses = (e, l1, s, dl)
        self._mark(timer, "loss")
        from .backward import K4_FORM
        common = (batch.rec.data_ptr(), idx.values.data_ptr(), idx.offsets.data_ptr(),
                  camera.width, camera.height, out.color.data_ptr(), out.depth.data_ptr(),
                  out.final_T.data_ptr(), out.n_considered.data_ptr(), out.ckpt.data_ptr(),
                  idx.ckpt_base.data_ptr(), grad_color.data_ptr(), _lib.ptr(gd), _lib.ptr(gt))
        ws = self.bwd_ws.get(camera.width, camera.height, idx.p_cap)
        if self.deterministic:  # slots + emission-order row sums overwrite grad2d
            det = (self.merges.data_ptr(), self.slots.data_ptr(), self.processed.data_ptr(),
                   *(t.data_ptr() for t in idx.det), idx.keys.data_ptr(), self.grad2d.shape[0],
                   self.scratch.totals.data_ptr(), self.grad2d.data_ptr())
            if K4_FORM in ("tiles", "regions"):
                _lib.check(self.lib.tsr_render_bwd_det(*common, *det, _lib.stream_handle()),
                           "tsr_render_bwd_det")
            else:
                _lib.check(self.lib.tsr_render_bwd_ws_det(
                    *common, *det, idx.p_cap, ws.data_ptr(), ws.numel(), _lib.stream_handle()),
                    "tsr_render_bwd_ws_det")
            self._grad2d_clean = False
            self._mark(timer, "backward")
            return e
        if not self._grad2d_clean:
            self.grad2d.zero_()
        self._grad2d_clean = False
        if update is not None and self._can_fuse_update():
            groups, scal = update
            s_ = self.scratch
            _lib.check(self.lib.tsr_render_bwd_adam(
                *common, self.grad2d.data_ptr(), self.merges.data_ptr(),
                _lib.ptr(self.tile_order), gaussians_struct(self.gset),
                camera_struct(camera, None, self.cfg.near), groups, _lib.ptr(scal),
                s_.source_ids.data_ptr(), s_.row_of_source.data_ptr(), s_.counts.data_ptr(),
                self.row_done.data_ptr(), self.skipped.data_ptr(), idx.overflow.data_ptr(),
                self.gated_steps.data_ptr(), e.data_ptr(), _lib.stream_handle()),
                "tsr_render_bwd_adam")
            self._updated = True
        elif self.regions is not None:
            from .backward import backward_regions_raw
            backward_regions_raw(batch.rec, idx.values, idx.offsets, camera.width, camera.height,
                                 out, idx.ckpt_base, self.regions, grad_color, gd, gt,
                                 self.grad2d, self.merges)
        elif K4_FORM in ("tiles", "regions"):
            _lib.check(self.lib.tsr_render_bwd_ordered(
                *common, self.grad2d.data_ptr(), self.merges.data_ptr(),
                _lib.ptr(self.tile_order), _lib.stream_handle()), "tsr_render_bwd_ordered")
        else:
            _lib.check(self.lib.tsr_render_bwd_ws(
                *common, self.grad2d.data_ptr(), self.merges.data_ptr(), idx.p_cap,
                ws.data_ptr(), ws.numel(), _lib.stream_handle()), "tsr_render_bwd_ws")
        self._mark(timer, "backward")
        return e

    def _publish_status(self) -> None:
        self.status_ovf_host.copy_(self.index.overflow, non_blocking=True)
        self.status_tot_host.copy_(self.scratch.totals, non_blocking=True)
        self.status_event = torch.cuda.Event()
        self.status_event.record()

    def _graph_key(self, camera: Camera, gt_image, depth_on: bool, depth_prior, depth_valid):
        return (camera.fx, camera.fy, camera.cx, camera.cy, camera.width, camera.height,
                camera.rotation.tobytes(), camera.translation.tobytes(), gt_image.data_ptr(),
                depth_on, _lib.ptr(depth_prior) if depth_on else 0,
                _lib.ptr(depth_valid) if depth_on else 0)

    def _graph_body(self, camera: Camera, gt_image, depth_on: bool, depth_prior, depth_valid):
        """The captured step: K1-K5 (K4b+K5 fused into K4 for SH 0) and the
        status publish; the per-step scalars are read from _scal_dev."""
        batch = self.forward(camera, None)
        groups = self.opt.groups_for_fused(self.gset.params(), None, advance=False)
        e = self.loss_and_backward(batch, camera, gt_image, None,
                                   self._scal_dev[15] if depth_on else 0.0,
                                   depth_prior if depth_on else None, depth_valid,
                                   update=(groups, self._scal_dev))
        if not self._updated:
            _lib.check(self.lib.tsr_preprocess_bwd_adam_ex(
                gaussians_struct(self.gset), camera_struct(camera, None, self.cfg.near),
                batch.rec.data_ptr(), batch.row_of_source.data_ptr(), self.grad2d.data_ptr(),
                groups, self._scal_dev.data_ptr(), None, self.skipped.data_ptr(),
                self.index.overflow.data_ptr(), self.gated_steps.data_ptr(), e.data_ptr(),
                _lib.stream_handle()), "tsr_preprocess_bwd_adam_ex")
        self.status_ovf_host.copy_(self.index.overflow, non_blocking=True)
        self.status_tot_host.copy_(self.scratch.totals, non_blocking=True)
        return e

    def _graph_step(self, camera: Camera, gt_image, depth_weight, depth_prior, depth_valid):
        cap = self.index.p_cap
        self._poll_status(camera)
        if self.index.p_cap != cap:  # capacity grew: the buffers moved
            self._graph_cache.clear()
        self.iteration += 1
        lr = {"positions": position_lr(self.pos_base_lr, self.iteration, self.cfg.max_iters)}
        descs = self.opt.groups_for_fused(self.gset.params(), lr)  # advances the step counts
        k = self._ring_k
        self._ring_k = (k + 1) % len(self._ring)
        if self._ring_ev[k] is not None:
            self._ring_ev[k].synchronize()  # that slot's copy has been consumed
        host = self._ring[k]
        for j, d in enumerate(descs):
            host[3 * j] = d.lr
            host[3 * j + 1] = d.bias_correction1
            host[3 * j + 2] = d.bias_correction2
        host[15] = float(depth_weight)
        self._scal_dev.copy_(host, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._ring_ev[k] = ev
        depth_on = depth_weight > 0.0 and depth_prior is not None
        key = self._graph_key(camera, gt_image, depth_on, depth_prior, depth_valid)
        entry = self._graph_cache.get(key)
        if entry is None:
            torch.cuda.current_stream().synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                e = self._graph_body(camera, gt_image, depth_on, depth_prior, depth_valid)
            entry = self._graph_cache[key] = (g, e)
        entry[0].replay()
        self._remember(camera, gt_image, depth_weight, depth_prior, depth_valid, None)
        self._grad2d_clean = self.gset.colors.shape[1] == 1
        self.status_event = torch.cuda.Event()
        self.status_event.record()
        self.last_camera = camera
        return entry[1]

    def step(self, camera: Camera, gt_image: torch.Tensor, timer=None,
             depth_weight: float = 0.0, depth_prior=None, depth_valid=None) -> torch.Tensor:
        """Run one step; returns the loss as a device scalar (no host sync)."""
        if self.graphs and timer is None and self.index is not None and self._grad2d_clean:
            return self._graph_step(camera, gt_image, depth_weight, depth_prior, depth_valid)
        if self.index is not None:
            self._poll_status(camera)
        e = self._eager_step(camera, gt_image, timer, depth_weight, depth_prior, depth_valid)
        self._remember(camera, gt_image, depth_weight, depth_prior, depth_valid,
                       self.last_losses)
        return e

    def _remember(self, camera, gt_image, depth_weight, depth_prior, depth_valid, outs):
        self._history.append((camera, gt_image, depth_weight, depth_prior, depth_valid,
                              self.iteration, outs))
        if len(self._history) > self.HISTORY:
            del self._history[0]

    def _eager_step(self, camera, gt_image, timer, depth_weight, depth_prior, depth_valid):
        self.iteration += 1
        batch = self.forward(camera, timer)
        lr = {"positions": position_lr(self.pos_base_lr, self.iteration, self.cfg.max_iters)}
        groups = self.opt.groups_for_fused(self.gset.params(), lr)
        e = self.loss_and_backward(batch, camera, gt_image, timer, depth_weight, depth_prior,
                                   depth_valid, update=(groups, None))
        if not self._updated:
            _lib.check(self.lib.tsr_preprocess_bwd_adam_ex(
                gaussians_struct(self.gset), camera_struct(camera, None, self.cfg.near),
                batch.rec.data_ptr(), batch.row_of_source.data_ptr(), self.grad2d.data_ptr(),
                groups, None, None, self.skipped.data_ptr(), self.index.overflow.data_ptr(),
                self.gated_steps.data_ptr(), e.data_ptr(), _lib.stream_handle()),
                "tsr_preprocess_bwd_adam_ex")
        self._grad2d_clean = self.gset.colors.shape[1] == 1
        self._mark(timer, "vjp_adam")
        self._publish_status()
        self.last_camera = camera
        return e

    def sync(self) -> None:
        """Wait for the queued steps and settle their status: an overflowed
        step is redone with a grown capacity before this returns."""
        torch.cuda.current_stream().synchronize()
        if self.index is not None and self.last_camera is not None:
            self._poll_status(self.last_camera)

    def kernels_per_step(self) -> int:
        """Our kernel launches per step: K1a, K1b; K2 (one persistent
        cooperative kernel); K3; loss (fwd, bwd + finalize); K4 (+ its two
        work-unit plan kernels); fused K4b+K5 (+ the row reduction in
        deterministic mode)."""
        from .backward import K4_FORM
        from .forward import TILE_ORDER
        return (2 + 1 + (1 if TILE_ORDER == "heavy" else 0) + 1 + 2 + 1
                + (2 if K4_FORM == "units" else 0)
                + 1 + (1 if self.deterministic else 0))

    def last_view(self):
        """(batch, TileIndex, RenderBuffers) views of the last step (synchronises)."""
        torch.cuda.current_stream().synchronize()
        overflow = int(self.index.overflow.item())
        if overflow:
            raise RuntimeError("pair capacity overflowed")
        m, p = (int(v) for v in self.scratch.totals.tolist())
        cam = self.last_camera
        s = self.scratch
        batch = SplatBatch(None, None, None, None, None, s.source_ids[:m], cam.width, cam.height,
                           _rec=s.rec[:m])
        tiles = TileIndex(self.index.keys[:p], self.index.values[:p], self.index.offsets,
                          cam.tiles_x, cam.tiles_y, self.index.ckpt_base)
        out = self.targets
        bufs = RenderBuffers(out.color, out.depth, out.final_T, out.n_contrib, out.n_considered,
                             np.asarray(self.cfg.background, float), out.ckpt,
                             self.index.ckpt_base, cam.tiles_x, cam.tiles_y)
        return batch, tiles, bufs


def phase_times(timer) -> dict:
    """Per-phase device milliseconds summed over the recorded steps."""
    out = {}
    evs = timer.get("_events", [])
    for (_, a), (name, b) in zip(evs, evs[1:]):
        if name == "start":
            continue
        out[name] = out.get(name, 0.0) + a.elapsed_time(b)
    return out


# --------------------------------------------------------------------------
# The training loop (trainer.py:255-395)


class TrainingDiverged(RuntimeError):
    def __init__(self, message, dump=None):
        super().__init__(message)
        self.dump = dump or {}


@dataclass
class TrainResult:
    gset: GaussianSet
    metrics: list
    delta: PoseDelta
    baked_total: PoseDelta
    iterations: int
    elapsed: float
    stop_reason: str  # completed | budget
    eval_split: str = "train"


def _mean_neighbour_distance(pts: np.ndarray, k: int = 3) -> np.ndarray:
    """Mean distance of every point to its k nearest other points (host,
    once per run; scipy's KD-tree, as the reference's trainer.py:147)."""
    from scipy.spatial import cKDTree
    dist, _ = cKDTree(pts).query(pts, k=k + 1, workers=-1)
    return dist[:, 1:].mean(axis=1)


def init_gaussians(scene, sh_degree: int = 0, init_opacity: float = 0.1) -> GaussianSet:
    """Seed one isotropic splat per point of the scene's cloud (trainer.py:137-
    160): radius = mean distance to the 3 nearest neighbours (floored at 1e-7;
    0.1 x extent for clouds of fewer than 4 points), DC colour = point colour /
    255, identity rotation, opacity `init_opacity`."""
    pts = np.array(scene.points, dtype=np.float64).reshape(-1, 3)
    count = pts.shape[0]
    if count == 0:
        raise ValueError("cannot initialize from an empty point cloud")
    if count < 4:
        radius = np.full(count, 0.1 * float(scene.extent))
    else:
        radius = np.maximum(_mean_neighbour_distance(pts), 1e-7)
    n_coeffs = (sh_degree + 1) ** 2
    colors = np.zeros((count, n_coeffs, 3))
    colors[:, 0] = np.asarray(scene.colors, dtype=np.float64) / 255.0
    log_r = np.log(radius)
    return GaussianSet(
        positions=pts,
        log_scales=np.stack([log_r, log_r, log_r], axis=1),
        rotations=np.tile(np.array([1.0, 0.0, 0.0, 0.0]), (count, 1)),
        opacity_logits=np.full(count, np.log(init_opacity) - np.log1p(-init_opacity)),
        colors=colors)


def evaluate(gset: GaussianSet, cameras, cfg: TrainConfig | None = None,
             delta: PoseDelta | None = None) -> float:
    """Mean PSNR of the renders against the cameras that carry ground truth
    (trainer.py:260-270); cameras without it are ignored."""
    scored = [cam for cam in cameras if cam.gt_image is not None]
    if not scored:
        raise ValueError("evaluate() needs at least one camera with a ground-truth image")
    cfg = TrainConfig() if cfg is None else cfg
    total = 0.0
    for cam in scored:
        color = render_view(gset, cam, cfg, delta, checkpoints=False).buffers.color
        total += losses.psnr(color, cam.gt_image)
    return total / len(scored)


def _densify_round(gset, scene, cfg, delta, rng, pool):
    """(s+, s-) of one density round through materialised Contributions
    (trainer.py:273-290): K views drawn from the pool, each rendered in
    scoring mode, its error mask and photometric error collected; the fused
    form below is what train() uses."""
    from . import density
    drawn = pool[rng.integers(0, len(pool), size=cfg.consistency_views)]
    per_view = {"masks": [], "pixels": [], "ids": [], "errors": []}
    for view in drawn:
        cam = scene.cameras[int(view)]
        vr = render_view(gset, cam, cfg, delta, checkpoints=False, scoring=True)
        contrib = vr.contributions
        per_view["masks"].append(density.error_mask(vr.buffers.color, cam.gt_image,
                                                    cfg.error_tau))
        per_view["pixels"].append(contrib.pixel_idx)
        per_view["ids"].append(vr.batch.source_ids[contrib.splat_rows])
        per_view["errors"].append(
            losses.photometric(vr.buffers.color, cam.gt_image, cfg.lambda_)[0].photometric)
    n = len(gset)
    return (density.score_densify(per_view["masks"], per_view["pixels"], per_view["ids"], n),
            density.score_prune(per_view["masks"], per_view["pixels"], per_view["ids"],
                                per_view["errors"], n))


def _densify_round_fused(gset, scene, cfg, delta, rng, pool, gt_dev):
    """The same scores with K3 scoring mode 3: per view one render, the error
    mask, and one masked-count render straight into per-row scores; no
    contribution lists.  Draws the same view ids from rng."""
    from . import density
    k = cfg.consistency_views
    view_ids = pool[rng.integers(0, len(pool), size=k)]
    n = len(gset)
    dev = _device()
    s_plus = torch.zeros(n, dtype=torch.float64, device=dev)
    raw = torch.zeros(n, dtype=torch.float64, device=dev)
    for v in view_ids:
        cam = scene.cameras[int(v)]
        vr = render_view(gset, cam, cfg, delta, checkpoints=False)
        gt = gt_dev[int(v)]
        e, _, _, _ = losses.photometric_device(vr.buffers.color, gt, cfg.lambda_)
        mask = density.error_mask(vr.buffers.color, gt, cfg.error_tau)
        counts = density.masked_row_counts(vr.batch, vr.tiles, cfg.background, mask)
        src = vr.batch.source_ids.long()
        c64 = counts.double()
        s_plus.index_add_(0, src, c64)
        raw.index_add_(0, src, e.double() * c64)
    return s_plus / max(k, 1), density._minmax(raw)


def train(scene, cfg: TrainConfig, *, ply_path=None, metrics_path=None, decisions_path=None,
          initial: GaussianSet | None = None, fused_scoring: bool = True) -> TrainResult:
    """The reference loop (trainer.py:293-395): view sampling, render, loss,
    backward, Adam, densify/prune cadence, pose bake cadence, PSNR cadence,
    wall-clock budget stop, PLY save.

    Without pose optimisation every iteration is one `TrainStep` (no host
    synchronisation; per-iteration losses stay on the device and are read
    at eval points, where the budget and divergence are also checked).  With
    pose optimisation the composable API path (render_view ->
    view_loss_and_grads -> _full_grads -> Adam) runs, as in the reference."""
    import time
    from pathlib import Path
    from . import density
    from .pose import bake, compose, identity_delta
    if not scene.cameras:
        raise ValueError("scene has no cameras")
    rng = np.random.default_rng(cfg.seed)
    gset = initial.copy() if initial is not None else init_gaussians(
        scene, cfg.sh_degree, cfg.init_opacity)
    holdout = set(int(i) for i in cfg.holdout_views)
    pool = np.array([i for i in range(len(scene.cameras)) if i not in holdout])
    if len(pool) == 0:
        raise ValueError("holdout_views leaves no training cameras")
    eval_cams = [scene.cameras[i] for i in sorted(holdout)] if holdout else scene.cameras
    opt = Adam({k: v for k, v in cfg.lrs.items() if k != "positions"})
    pos_base_lr = cfg.lrs.get("positions", 1.6e-4 * scene.extent)
    delta = identity_delta() if cfg.pose_opt else None
    baked_total = identity_delta()
    gt_dev = [as_device_f32(c.gt_image) if c.gt_image is not None else None
              for c in scene.cameras]
    prior_dev = [as_device_f32(c.depth_prior) if c.depth_prior is not None else None
                 for c in scene.cameras]
    valid_dev = [(c.depth_valid.to(_device()).bool() if isinstance(c.depth_valid, torch.Tensor)
                  else torch.as_tensor(np.asarray(c.depth_valid), device=_device()).bool())
                 if c.depth_valid is not None else None for c in scene.cameras]
    # cfg.deterministic (default True, like the reference) selects K4's
    # deterministic merge: the same seed gives bitwise-identical metrics
    stepper = None if cfg.pose_opt else TrainStep(gset, cfg, extent=scene.extent, optimizer=opt,
                                                  deterministic=cfg.deterministic)
    train_cams = [scene.cameras[int(i)] for i in pool]
    pose_t = {k: torch.zeros((1, 3), dtype=torch.float32, device=_device())
              for k in ("pose_rot", "pose_trans")}
    metrics, pending, decision_rows = [], [], []
    stop_reason = "completed"
    start = time.perf_counter()
    if stepper is not None:
        # pair capacity for the largest training view (one host read; on the
        # budget clock, like the reference's first-iteration setup)
        stepper.reserve(train_cams)
    iteration = 0

    def flush():
        """Read the pending device losses; divergence check."""
        if not pending:
            return
        vals = torch.stack([torch.stack([e, l1, s, d]) for _, e, l1, s, d in pending]).cpu()
        for (it, *_), row in zip(pending, vals.tolist()):
            if not np.isfinite(row[0]):
                # the fused update skipped this step on the device (loss
                # guard), so the set is the one that produced the loss
                from .scene import validate
                dump = {"iteration": it, "loss": row[0], "l1": row[1], "ssim": row[2],
                        "invariant_report": validate(gset)}
                if ply_path:
                    Path(ply_path).with_suffix(".diverged.json").write_text(
                        json.dumps(dump, indent=2))
                raise TrainingDiverged(f"non-finite loss at iteration {it}", dump)
            metrics.append({"iter": it, "l1": row[1], "ssim": row[2], "depth_loss": row[3],
                            "total": row[0], "psnr": np.nan})
        pending.clear()

    zero = torch.zeros((), device=_device())
    while iteration < cfg.max_iters:
        iteration += 1
        v = int(pool[rng.integers(0, len(pool))])
        cam = scene.cameras[v]
        depth_weight = (losses.depth_weight_schedule(iteration - 1, cfg.max_iters,
                                                     cfg.depth_weight0)
                        if cfg.depth_supervision else 0.0)
        if stepper is not None:
            stepper.iteration = iteration - 1
            stepper.step(cam, gt_dev[v], depth_weight=depth_weight, depth_prior=prior_dev[v],
                         depth_valid=valid_dev[v])
            e, l1, s, dl = stepper.last_losses
            pending.append((iteration, e, l1, s, dl if dl is not None else zero))
        else:
            vr = render_view(gset, cam, cfg, delta)
            report, g2 = view_loss_and_grads(cam, cfg, vr, depth_weight)
            grads = _full_grads(gset, cam, cfg, delta, vr, g2)
            opt.step(gset.params(), {k: grads[k] for k in gset.params()},
                     {"positions": position_lr(pos_base_lr, iteration, cfg.max_iters)})
            pose_t["pose_rot"].copy_(torch.as_tensor(delta.rot_vec).reshape(1, 3))
            pose_t["pose_trans"].copy_(torch.as_tensor(delta.trans).reshape(1, 3))
            opt.step(pose_t, {k: torch.as_tensor(np.asarray(grads[k], np.float32)).reshape(1, 3)
                              for k in pose_t})
            delta.rot_vec[:] = pose_t["pose_rot"].double().cpu().numpy().reshape(3)
            delta.trans[:] = pose_t["pose_trans"].double().cpu().numpy().reshape(3)
            delta.steps_since_bake += 1
            t = lambda x: torch.tensor(float(x), device=_device())  # noqa: E731
            pending.append((iteration, t(report.total), t(report.l1), t(report.ssim),
                            t(report.depth_loss)))

        if (cfg.densify and cfg.densify_start <= iteration < cfg.densify_end
                and iteration % cfg.densify_interval == 0):
            flush()
            if fused_scoring:
                s_plus, s_minus = _densify_round_fused(gset, scene, cfg, delta, rng, pool, gt_dev)
            else:
                s_plus, s_minus = _densify_round(gset, scene, cfg, delta, rng, pool)
            threshold = cfg.scale_split_threshold_frac * scene.extent
            gset, decisions = density.apply_decisions(gset, s_plus, s_minus, cfg.theta_plus,
                                                      cfg.theta_minus, threshold, rng,
                                                      min_splats=cfg.min_splats)
            opt.resize(decisions)
            c = decisions.counts()
            decision_rows.append({"iter": iteration, "clones": c["clone"], "splits": c["split"],
                                  "prunes": c["prune"], "total": len(gset)})
            if stepper is not None:
                stepper = TrainStep(gset, cfg, extent=scene.extent, optimizer=opt,
                                    deterministic=cfg.deterministic)
                stepper.reserve(train_cams)

        if cfg.pose_opt and delta.steps_since_bake >= cfg.pose_bake_interval:
            baked = bake(delta, scene.cameras)
            baked_total = compose(baked_total, baked)
            opt.reset_group("pose_rot")
            opt.reset_group("pose_trans")

        if iteration % cfg.eval_interval == 0 or iteration == cfg.max_iters:
            flush()
            metrics[-1]["psnr"] = evaluate(gset, eval_cams, cfg, delta)
        if iteration % 32 == 0 or iteration == 1 or iteration == cfg.max_iters:
            # bound the launch queue so host time ~ device time (and the
            # first iteration's budget check sees its device time, like the
            # reference's synchronous step)
            torch.cuda.synchronize()
        if time.perf_counter() - start > cfg.budget_seconds:
            stop_reason = "budget"
            break
    flush()
    torch.cuda.synchronize()
    elapsed = time.perf_counter() - start
    result = TrainResult(gset=gset, metrics=metrics, delta=delta or identity_delta(),
                         baked_total=baked_total, iterations=iteration, elapsed=elapsed,
                         stop_reason=stop_reason,
                         eval_split="holdout" if holdout else "train")
    if ply_path:
        from .ingest import write_ply
        write_ply(gset, ply_path)
    if metrics_path:
        write_metrics_csv(metrics_path, metrics, eval_split=result.eval_split)
    if decisions_path:
        write_decisions_csv(decisions_path, decision_rows)
    return result


def write_metrics_csv(path, metrics, eval_split="train") -> None:
    with open(path, "w") as fh:
        fh.write(f"# eval split: {eval_split}\n")
        fh.write("iter,l1,ssim,depth_loss,total,psnr\n")
        for row in metrics:
            psnr = "" if np.isnan(row["psnr"]) else f"{row['psnr']:.6f}"
            fh.write(f"{row['iter']},{row['l1']:.8f},{row['ssim']:.8f},"
                     f"{row['depth_loss']:.8f},{row['total']:.8f},{psnr}\n")


def write_decisions_csv(path, rows) -> None:
    with open(path, "w") as fh:
        fh.write("iter,clones,splits,prunes,total\n")
        for row in rows:
            fh.write(f"{row['iter']},{row['clones']},{row['splits']},"
                     f"{row['prunes']},{row['total']}\n")
