"""View-parallel data parallelism over NCCL.

Gaussians are replicated; each rank rasterizes its own camera views (K1-K4,
K4b into one flat gradient buffer), the flat buffer is summed across ranks
with ONE allreduce per step, and every rank applies the identical Adam update
(K5), so replicas stay bit-identical.  `deterministic=True` replaces the
NCCL sum by an all-gather + fixed rank-order sum, making the result
independent of the reduction tree (bitwise-equal params for any N with the
same view set)."""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib
from .optim import Adam, SPLAT_GROUPS, position_lr
from .projection import camera_struct, gaussians_struct
from .trainer import TrainConfig, TrainStep


def shard_views(n_views: int, world: int, rank: int) -> list[int]:
    """Contiguous, balanced split of a camera batch across ranks."""
    base, rem = divmod(n_views, world)
    start = rank * base + min(rank, rem)
    return list(range(start, start + base + (1 if rank < rem else 0)))


def flat_grad_views(flat: torch.Tensor, gset) -> dict:
    """Per-group (N, ...) views into one flat gradient buffer, in optimizer
    group order, so one collective moves every gradient."""
    out, off = {}, 0
    for name, p in gset.params().items():
        n = p.numel()
        out[name] = flat[off: off + n].view_as(p)
        off += n
    return out


def grad_numel(gset) -> int:
    return sum(p.numel() for p in gset.params().values())


def allreduce_grads(flat: torch.Tensor, group=None, deterministic: bool = False) -> torch.Tensor:
    """Sum the flat gradient buffer over ranks (in place); a no-op without a
    process group (one GPU)."""
    if not dist.is_available() or not dist.is_initialized():
        return flat
    world = dist.get_world_size(group)
    if world == 1:
        return flat
    if not deterministic:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
        return flat
    parts = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(parts, flat, group=group)
    acc = parts[0].clone()
    for p in parts[1:]:
        acc += p
    flat.copy_(acc)
    return flat


class ViewParallelStep(TrainStep):
    """One optimizer step over this rank's views + an allreduce."""

    def __init__(self, gset, cfg: TrainConfig, extent: float = 4.0, group=None,
                 deterministic: bool = False):
        super().__init__(gset, cfg, extent)
        self.group = group
        self.deterministic = deterministic
        self.flat = torch.zeros(grad_numel(gset), dtype=torch.float32, device="cuda")
        self.grads = flat_grad_views(self.flat, gset)

    def kernels_per_step(self, views: int = 1) -> int:
        """Per view: K1-K4 + K4b; then one K5 (the NCCL allreduce is not ours)."""
        return views * (super().kernels_per_step() - 1 + 1) + 1

    def step_views(self, cameras, gts, timer=None) -> torch.Tensor:
        if self.index is not None and cameras:
            self._poll_status(cameras[0])
        self.iteration += 1
        total = None
        for k, (camera, gt) in enumerate(zip(cameras, gts)):
            batch = self.forward(camera, timer)
            e = self.loss_and_backward(batch, camera, gt, timer)
            g = self.grads
            _lib.check(self.lib.tsr_preprocess_bwd(
                gaussians_struct(self.gset), camera_struct(camera, None, self.cfg.near),
                batch.rec.data_ptr(), batch.row_of_source.data_ptr(), self.grad2d.data_ptr(),
                g["positions"].data_ptr(), g["log_scales"].data_ptr(), g["rotations"].data_ptr(),
                g["opacity_logits"].data_ptr(), g["colors"].data_ptr(), None, 1 if k else 0,
                _lib.stream_handle()), "tsr_preprocess_bwd")
            total = e if total is None else total + e
            self._publish_status()
            self.last_camera = camera
        if not cameras:
            self.flat.zero_()
        self._mark(timer, "vjp")
        allreduce_grads(self.flat, self.group, self.deterministic)
        self._mark(timer, "allreduce")
        lr = {"positions": position_lr(self.pos_base_lr, self.iteration, self.cfg.max_iters)}
        self.opt.step_async(self.gset.params(), self.grads, lr)
        self._mark(timer, "adam")
        return total
