"""View-parallel data parallelism over NCCL.

Gaussians are replicated; each rank rasterizes its own camera views (K1-K4,
K4b into one flat gradient buffer), the flat buffer is summed across ranks
with ONE allreduce per step, and every rank applies the identical Adam update
(K5), so replicas stay bit-identical.  `deterministic=True` replaces the
NCCL sum by an all-gather + fixed rank-order sum, making the result
independent of the reduction tree: bitwise reproducible for a fixed N and
view assignment (each rank first sums its own views locally, so a different
N reassociates those sums and agrees to FP32 tolerance, not bitwise).

`sharded=True` is the ZeRO-1 form of the same step (the
B200 variant): per group, a reduce-scatter gives rank r the summed
gradient of its row shard [r R, (r + 1) R) (R = ceil(N / G)), K5 updates
only that shard with shard-sized moments (Adam's work and its m, v memory
drop G-fold), and an all-gather of the updated rows makes the parameters
whole again on every rank.  Same bytes on the wire as the allreduce; the
result is bitwise the replicated step's (Adam is row-local)."""

from __future__ import annotations

import ctypes
import os

import torch
import torch.distributed as dist

from . import _lib
from .optim import BETA1, BETA2, Adam, SPLAT_GROUPS, position_lr
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


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int, int]:
    """This rank's optimizer row shard [s, e) and the padded shard size R
    (every group splits its rows the same way; the last shard may be short)."""
    r = -(-n // world) if n else 0
    s = min(rank * r, n)
    return s, min(s + r, n), r


def padded_grad_views(flat: torch.Tensor, gset, rows: int) -> dict:
    """Per-group (rows, ...) views into one flat buffer, rows >= N (the
    padding rows stay zero), in optimizer group order."""
    out, off = {}, 0
    for name, p in gset.params().items():
        shape = (rows,) + tuple(p.shape[1:])
        n = rows * (p.numel() // max(p.shape[0], 1))
        out[name] = flat[off: off + n].view(shape)
        off += n
    return out


def _world_rank(group):
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def reduce_scatter_rows(full: torch.Tensor, out: torch.Tensor, group=None,
                        deterministic: bool = False) -> torch.Tensor:
    """out (R, ...) = sum over ranks of rows [rank R, (rank + 1) R) of full
    (G R, ...).  NCCL: one reduce_scatter_tensor; gloo (no reduce-scatter)
    and deterministic mode: the allreduce forms above, then this rank's rows."""
    world, rank = _world_rank(group)
    r = out.shape[0]
    if world == 1:
        return out.copy_(full[:r])
    if not deterministic and dist.get_backend(group) == "nccl":
        dist.reduce_scatter_tensor(out, full, group=group)
        return out
    summed = allreduce_grads(full.clone(), group, deterministic)
    return out.copy_(summed[rank * r:(rank + 1) * r])


def all_gather_rows(shard: torch.Tensor, full: torch.Tensor, group=None) -> torch.Tensor:
    """full (G R, ...) = the ranks' (R, ...) shards in rank order."""
    world, _ = _world_rank(group)
    if world == 1:
        return full[:shard.shape[0]].copy_(shard)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(full, shard, group=group)
    else:
        dist.all_gather(list(full.chunk(world)), shard, group=group)
    return full


class ZeroAdam:
    """ZeRO-1 Adam over a row shard (optim.py:60-88 semantics per row): this
    rank owns the moments of rows [s, e) of every group; lr, bias
    corrections and the per-group step counts follow Adam exactly."""

    def __init__(self, gset, world: int, rank: int, lrs: dict | None = None):
        self.adam = Adam(lrs)
        self.s, self.e, self.rows = shard_rows(len(gset), world, rank)
        self.m = {k: torch.zeros((self.rows,) + tuple(p.shape[1:]), dtype=torch.float32,
                                 device="cuda") for k, p in gset.params().items()}
        self.v = {k: torch.zeros_like(t) for k, t in self.m.items()}
        self.steps = {k: 0 for k in self.m}

    def step_async(self, params: dict, grad_shards: dict, lr_overrides=None) -> torch.Tensor:
        lib = _lib.load()
        descs = []
        n = self.e - self.s
        for name, p in params.items():
            self.steps[name] += 1
            t = self.steps[name]
            width = p.numel() // max(p.shape[0], 1)
            d = _lib.AdamGroup_t()
            d.param = p.data_ptr() + 4 * self.s * width
            d.grad = grad_shards[name].data_ptr()
            d.exp_avg = self.m[name].data_ptr()
            d.exp_avg_sq = self.v[name].data_ptr()
            d.rows = n
            d.width = width
            d.renormalize = 1 if name == "rotations" else 0
            d.lr = (lr_overrides or {}).get(name, self.adam.lrs.get(name, 1e-3))
            d.bias_correction1 = 1.0 - BETA1 ** t
            d.bias_correction2 = 1.0 - BETA2 ** t
            descs.append(d)
        counter = self.adam._counter()
        if n > 0:
            arr = (_lib.AdamGroup_t * len(descs))(*descs)
            _lib.check(lib.tsr_adam_step(arr, len(descs), counter.data_ptr(),
                                         _lib.stream_handle()), "tsr_adam_step")
        return counter


def share_peer_tensors(tensors: list, group=None) -> list:
    """Every rank's `tensors`, opened in this process: CUDA IPC handles
    (torch.multiprocessing's rebuild path) exchanged with one all_gather_object.
    Returns [rank][i] tensors aliasing the peers' device memory (this rank's
    own entries are the originals)."""
    from torch.multiprocessing.reductions import reduce_tensor
    world, rank = _world_rank(group)
    if world == 1:
        return [list(tensors)]
    mine = [reduce_tensor(t) for t in tensors]
    everyone = [None] * world
    dist.all_gather_object(everyone, mine, group=group)
    out = []
    for q, items in enumerate(everyone):
        if q == rank:
            out.append(list(tensors))
        else:
            out.append([fn(*args) for fn, args in items])
    return out


class PeerZeroUpdate:
    """ZeRO-1 fused over peer memory (tsr_zero1_peer_adam): one kernel per
    rank reads every rank's gradient rows of its shard through CUDA IPC
    mappings, sums them in rank order, runs Adam with shard moments and
    stores the updated rows into every rank's parameters.  Two host barriers
    order it: all gradients complete before any rank reads them; all
    updates complete before the parameters (or gradient buffers) are
    touched again.  Fixed N (no densification in this mode)."""

    def __init__(self, gset, grads: dict, zero: ZeroAdam, world: int, group=None):
        self.world, self.group, self.zero = world, group, zero
        names = list(gset.params())
        self.names = names
        local = [grads[n] for n in names] + [gset.params()[n] for n in names]
        peers = share_peer_tensors(local, group)
        self._peers = peers  # keep the mappings alive
        ng = len(names)
        ptr_g = [peers[q][k].data_ptr() for q in range(world) for k in range(ng)]
        ptr_p = [peers[q][ng + k].data_ptr() for q in range(world) for k in range(ng)]
        self.peer_grads = (ctypes.c_void_p * len(ptr_g))(*ptr_g)
        self.peer_params = (ctypes.c_void_p * len(ptr_p))(*ptr_p)

    def step(self, params: dict, lr_overrides=None) -> None:
        lib = _lib.load()
        z = self.zero
        descs = []
        for name in self.names:
            p = params[name]
            z.steps[name] += 1
            t = z.steps[name]
            d = _lib.AdamGroup_t()
            d.param = p.data_ptr()
            d.grad = None
            d.exp_avg = z.m[name].data_ptr()
            d.exp_avg_sq = z.v[name].data_ptr()
            d.rows = p.shape[0]
            d.width = p.numel() // max(p.shape[0], 1)
            d.renormalize = 1 if name == "rotations" else 0
            d.lr = (lr_overrides or {}).get(name, z.adam.lrs.get(name, 1e-3))
            d.bias_correction1 = 1.0 - BETA1 ** t
            d.bias_correction2 = 1.0 - BETA2 ** t
            descs.append(d)
        arr = (_lib.AdamGroup_t * len(descs))(*descs)
        _barrier(self.group)  # every rank's gradients are complete
        _lib.check(lib.tsr_zero1_peer_adam(arr, len(descs), self.world, self.peer_grads,
                                           self.peer_params, z.s, z.e,
                                           z.adam._counter().data_ptr(), _lib.stream_handle()),
                   "tsr_zero1_peer_adam")
        _barrier(self.group)  # every rank's rows are stored everywhere


def _barrier(group):
    torch.cuda.current_stream().synchronize()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.barrier(group=group)


class ChunkedGrads:
    """Chunk-major flat gradient buffer for the overlapped exchange: the
    Gaussian rows are split into `chunks` ranges and each range's five group
    gradients are contiguous, so one collective moves one chunk.  K4b writes
    a chunk through row-offset views of the set (no kernel change), Adam
    updates it through row-offset descriptors (Adam is row-local)."""

    def __init__(self, gset, chunks: int):
        n = len(gset)
        self.bounds = [n * c // chunks for c in range(chunks + 1)]
        widths = [p.numel() // max(p.shape[0], 1) for p in gset.params().values()]
        self.names = list(gset.params())
        self.widths = dict(zip(self.names, widths))
        self.row_floats = sum(widths)
        self.flat = torch.zeros(n * self.row_floats, dtype=torch.float32, device="cuda")
        # chunk c starts at row_floats * bounds[c]; inside it group g starts at
        # rows_c * (sum of the widths before g)
        self.seg = []
        for c in range(chunks):
            r0, r1 = self.bounds[c], self.bounds[c + 1]
            base, off, seg = self.row_floats * r0, 0, {}
            for name, w in zip(self.names, widths):
                seg[name] = base + off
                off += (r1 - r0) * w
            self.seg.append(seg)

    def chunk(self, c: int) -> torch.Tensor:
        r0, r1 = self.bounds[c], self.bounds[c + 1]
        return self.flat[self.row_floats * r0: self.row_floats * r1]

    def ptr(self, c: int, name: str) -> int:
        return self.flat.data_ptr() + 4 * self.seg[c][name]

    def group_views(self) -> dict:
        """Per-group (N, ...) gradients gathered from the chunks (tests)."""
        out = {}
        for name in self.names:
            w = self.widths[name]
            parts = [self.flat[self.seg[c][name]: self.seg[c][name] +
                               (self.bounds[c + 1] - self.bounds[c]) * w]
                     for c in range(len(self.seg))]
            out[name] = torch.cat(parts).view(-1, w)
        return out


class ViewParallelStep(TrainStep):
    """One optimizer step over this rank's views + an allreduce (or, with
    sharded=True, reduce-scatter -> K5 on the row shard -> all-gather).

    With `chunks` > 1 (default 4 at N > 1 in the replicated mode) the last
    view's K4b runs per Gaussian-row chunk and each chunk's gradient is
    summed (one NCCL allreduce) and Adam-updated on a communication stream
    while K4b computes the next chunk, so the exchange overlaps the tail of
    the step."""

    def __init__(self, gset, cfg: TrainConfig, extent: float = 4.0, group=None,
                 deterministic: bool = False, sharded: bool = False, peer: bool = False,
                 chunks: int | None = None, force_collectives: bool = False,
                 graphs: bool = False):
        super().__init__(gset, cfg, extent)
        # CUDA-graph replay of the chunked step (after one eager step)
        self.graphs = graphs
        self.graph_error = None
        self._warm = False
        self.group = group
        self.deterministic = deterministic
        self.sharded = sharded or peer
        self.peer = None
        # collectives also at world size 1 (exercises the NCCL path on one GPU)
        self.force_collectives = force_collectives
        world, _ = _world_rank(group)
        if chunks is None:
            chunks = int(os.environ.get("TSR_VP_CHUNKS", 4 if world > 1 else 1))
        self.chunks = 1 if self.sharded else max(1, chunks)
        self.cgrads = None
        self.comm_stream = None
        if peer:  # fused ZeRO-1 over peer memory (tsr_zero1_peer_adam)
            world, rank = _world_rank(group)
            self.zero = ZeroAdam(gset, world, rank, self.opt.lrs)
            self.flat = torch.zeros(grad_numel(gset), dtype=torch.float32, device="cuda")
            self.grads = flat_grad_views(self.flat, gset)
            self.peer = PeerZeroUpdate(gset, self.grads, self.zero, world, group)
        elif sharded:
            world, rank = _world_rank(group)
            self.zero = ZeroAdam(gset, world, rank, self.opt.lrs)
            rows = self.zero.rows * world
            self.flat = torch.zeros(rows * sum(p.numel() // max(p.shape[0], 1)
                                               for p in gset.params().values()),
                                    dtype=torch.float32, device="cuda")
            self.grads = padded_grad_views(self.flat, gset, rows)
            self.grad_shards = {k: torch.zeros_like(t) for k, t in self.zero.m.items()}
            self.param_shards = {k: torch.zeros_like(t) for k, t in self.zero.m.items()}
            self.param_full = {k: torch.zeros_like(g) for k, g in self.grads.items()}
        elif self.chunks > 1:
            self.cgrads = ChunkedGrads(gset, self.chunks)
            self.flat = self.cgrads.flat
            self.grads = None
            self.comm_stream = torch.cuda.Stream()
            self._chunk_ev = [torch.cuda.Event() for _ in range(self.chunks)]
        else:
            self.flat = torch.zeros(grad_numel(gset), dtype=torch.float32, device="cuda")
            self.grads = flat_grad_views(self.flat, gset)

    # -------------------------------------------------- chunked exchange ---
    def _chunk_struct(self, c: int):
        """The set's rows [r0, r1) as a K4b input (row-offset pointers)."""
        r0, r1 = self.cgrads.bounds[c], self.cgrads.bounds[c + 1]
        g = gaussians_struct(self.gset)
        for name in ("positions", "log_scales", "rotations", "opacity_logits", "colors"):
            setattr(g, name, getattr(g, name) + 4 * r0 * self.cgrads.widths[name])
        g.n = r1 - r0
        return g

    def _vjp_chunk(self, camera, batch, c: int, accumulate: bool) -> None:
        r0 = self.cgrads.bounds[c]
        cg = self.cgrads
        _lib.check(self.lib.tsr_preprocess_bwd(
            self._chunk_struct(c), camera_struct(camera, None, self.cfg.near),
            batch.rec.data_ptr(), batch.row_of_source.data_ptr() + 4 * r0,
            self.grad2d.data_ptr(), cg.ptr(c, "positions"), cg.ptr(c, "log_scales"),
            cg.ptr(c, "rotations"), cg.ptr(c, "opacity_logits"), cg.ptr(c, "colors"), None,
            1 if accumulate else 0, _lib.stream_handle()), "tsr_preprocess_bwd")

    def _adam_chunk(self, c: int, descs: dict, stream, scal_dev=None) -> None:
        """K5 on rows [r0, r1) of every group (the step's lr / bias
        corrections -- by value, or from `scal_dev` under graph replay --
        gradient from chunk c)."""
        r0, r1 = self.cgrads.bounds[c], self.cgrads.bounds[c + 1]
        arr = (_lib.AdamGroup_t * len(descs))()
        for j, (name, d) in enumerate(descs.items()):
            w = self.cgrads.widths[name]
            e = arr[j]
            e.param = d.param + 4 * r0 * w
            e.grad = self.cgrads.ptr(c, name)
            e.exp_avg = d.exp_avg + 4 * r0 * w
            e.exp_avg_sq = d.exp_avg_sq + 4 * r0 * w
            e.rows = r1 - r0
            e.width = w
            e.renormalize = d.renormalize
            e.lr = d.lr
            e.bias_correction1 = d.bias_correction1
            e.bias_correction2 = d.bias_correction2
        if scal_dev is not None:
            _lib.check(self.lib.tsr_adam_step_dev(
                arr, len(descs), scal_dev.data_ptr(), len(descs), self.opt._counter().data_ptr(),
                ctypes.c_void_p(stream.cuda_stream)), "tsr_adam_step_dev")
        else:
            _lib.check(self.lib.tsr_adam_step(arr, len(descs), self.opt._counter().data_ptr(),
                                              ctypes.c_void_p(stream.cuda_stream)),
                       "tsr_adam_step")

    def _reduce_chunk(self, c: int) -> None:
        """Sum chunk c over ranks: one NCCL allreduce, or (deterministic) an
        all-gather + rank-order sum, bitwise independent of the tree."""
        if not self._collective():
            return
        chunk = self.cgrads.chunk(c)
        if self.deterministic:
            world, _ = _world_rank(self.group)
            parts = [torch.empty_like(chunk) for _ in range(world)]
            dist.all_gather(parts, chunk, group=self.group)
            acc = parts[0].clone()
            for q in parts[1:]:
                acc += q
            chunk.copy_(acc)
        else:
            dist.all_reduce(chunk, op=dist.ReduceOp.SUM, group=self.group)

    def _collective(self) -> bool:
        world, _ = _world_rank(self.group)
        return world > 1 or (self.force_collectives and dist.is_available()
                             and dist.is_initialized())

    def _step_views_chunked(self, cameras, gts, timer, descs=None, scal_dev=None) -> torch.Tensor:
        total = None
        main = torch.cuda.current_stream()
        if descs is None:
            lr = {"positions": position_lr(self.pos_base_lr, self.iteration, self.cfg.max_iters)}
            # the step's descriptors (advance the group step counts once)
            descs = {name: self.opt._group(name, p, None, lr)
                     for name, p in self.gset.params().items()}
        if not cameras:
            self.flat.zero_()
        last = len(cameras) - 1
        for k, (camera, gt) in enumerate(zip(cameras, gts)):
            batch = self.forward(camera, timer)
            e = self.loss_and_backward(batch, camera, gt, timer)
            total = e if total is None else total + e
            if torch.cuda.is_current_stream_capturing():  # copy nodes only
                self.status_ovf_host.copy_(self.index.overflow, non_blocking=True)
                self.status_tot_host.copy_(self.scratch.totals, non_blocking=True)
            else:
                self._publish_status()
            self.last_camera = camera
            for c in range(self.chunks):
                self._vjp_chunk(camera, batch, c, accumulate=k > 0)
                if k == last:  # exchange + update chunk c while K4b runs chunk c + 1
                    self._chunk_ev[c].record(main)
                    with torch.cuda.stream(self.comm_stream):
                        self.comm_stream.wait_event(self._chunk_ev[c])
                        self._reduce_chunk(c)
                        self._adam_chunk(c, descs, self.comm_stream, scal_dev)
        if cameras:
            done = torch.cuda.Event()
            done.record(self.comm_stream)
            main.wait_event(done)
        else:
            for c in range(self.chunks):
                with torch.cuda.stream(self.comm_stream):
                    self._reduce_chunk(c)
                    self._adam_chunk(c, descs, self.comm_stream, scal_dev)
            done = torch.cuda.Event()
            done.record(self.comm_stream)
            main.wait_event(done)
        self._mark(timer, "vjp_allreduce_adam")
        return total

    def kernels_per_step(self, views: int = 1) -> int:
        """Per view: K1-K4 + K4b (one per row chunk); then K5 (one per row
        chunk).  The NCCL collectives are not ours."""
        return views * (super().kernels_per_step() - 1 + self.chunks) + self.chunks

    def _recover_overflow(self, camera) -> None:
        # the view batch is reserved up front (step_views), and this path's
        # update (allreduce + K5) is not gated: an overflow here means the
        # 1.5x headroom was outgrown mid-run
        raise RuntimeError(f"pair capacity {self.index.p_cap} overflowed in the view-parallel "
                           "step; reserve() a larger capacity for the view batch")

    def _graph_step_views(self, cameras, gts) -> torch.Tensor:
        """The chunked step replayed as ONE CUDA graph: every view's K1-K4b,
        the per-chunk NCCL allreduces and Adam updates on the communication
        stream (forked from and joined back into the capture stream), and
        the status copies.  The step's Adam scalars reach the captured K5
        launches from device memory (pinned ring + copy, as TrainStep)."""
        cap = self.index.p_cap
        self._poll_status(cameras[0])
        if self.index.p_cap != cap:
            self._graph_cache.clear()
        self.iteration += 1
        lr = {"positions": position_lr(self.pos_base_lr, self.iteration, self.cfg.max_iters)}
        descs = {name: self.opt._group(name, p, None, lr)
                 for name, p in self.gset.params().items()}
        k = self._ring_k
        self._ring_k = (k + 1) % len(self._ring)
        if self._ring_ev[k] is not None:
            self._ring_ev[k].synchronize()
        host = self._ring[k]
        for j, d in enumerate(descs.values()):
            host[3 * j], host[3 * j + 1], host[3 * j + 2] = (d.lr, d.bias_correction1,
                                                             d.bias_correction2)
        self._scal_dev.copy_(host, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._ring_ev[k] = ev
        key = tuple(self._graph_key(c, g, False, None, None) for c, g in zip(cameras, gts))
        entry = self._graph_cache.get(key)
        if entry is None:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(g):
                    e = self._step_views_chunked(cameras, gts, None, descs=descs,
                                                 scal_dev=self._scal_dev)
            except RuntimeError as exc:
                # a communicator that cannot be captured: run this (and every
                # later) step eagerly instead -- same kernels, same result
                import sys
                print(f"[tilesplat_b200] CUDA-graph capture of the view-parallel step failed "
                      f"({exc}); continuing with eager launches", file=sys.stderr)
                self.graphs = False
                self.graph_error = str(exc)[:200]
                torch.cuda.synchronize()
                return self._step_views_chunked(cameras, gts, None, descs=descs,
                                                scal_dev=self._scal_dev)
            entry = self._graph_cache[key] = (g, e)
        entry[0].replay()
        self.status_event = torch.cuda.Event()
        self.status_event.record()
        self.last_camera = cameras[-1]
        return entry[1]

    def step_views(self, cameras, gts, timer=None) -> torch.Tensor:
        if self.index is None and cameras:
            self.reserve(cameras)  # pair capacity for the largest view of the batch
        if (self.graphs and timer is None and self.cgrads is not None and cameras
                and self._warm):
            return self._graph_step_views(cameras, gts)
        if self.index is not None and cameras:
            self._poll_status(cameras[0])
        self.iteration += 1
        if self.cgrads is not None:
            out = self._step_views_chunked(cameras, gts, timer)
            self._warm = True  # the collectives ran once eagerly (NCCL warm-up)
            return out
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
        lr = {"positions": position_lr(self.pos_base_lr, self.iteration, self.cfg.max_iters)}
        if self.peer is not None:
            self.peer.step(self.gset.params(), lr)
            self._mark(timer, "adam")
            return total
        if self.sharded:
            return self._sharded_update(lr, timer, total)
        if self.force_collectives and _world_rank(self.group)[0] == 1 and dist.is_initialized():
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group)
        else:
            allreduce_grads(self.flat, self.group, self.deterministic)
        self._mark(timer, "allreduce")
        self.opt.step_async(self.gset.params(), self.grads, lr)
        self._mark(timer, "adam")
        return total

    def _sharded_update(self, lr, timer, total):
        params = self.gset.params()
        for name in params:
            reduce_scatter_rows(self.grads[name], self.grad_shards[name], self.group,
                                self.deterministic)
        self._mark(timer, "allreduce")
        self.zero.step_async(params, self.grad_shards, lr)
        self._mark(timer, "adam")
        s, e = self.zero.s, self.zero.e
        for name, p in params.items():
            shard = self.param_shards[name]
            shard[:e - s].copy_(p[s:e])
            all_gather_rows(shard, self.param_full[name], self.group)
            p.copy_(self.param_full[name][:p.shape[0]])
        self._mark(timer, "allgather")
        return total
