"""Adam on the B200 (reference: tilesplat/optim.py).

`Adam.step` launches K5 (csrc/vjp_adam.cu) once for all groups: dense
bias-corrected update of every row, rows with a non-finite gradient skipped
(moments and parameters untouched) and counted, rotation rows renormalised
(optim.py:60-88).  Step counters and bias corrections stay on the host in
float64 (they are per-group scalars).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

BETA1 = 0.9
BETA2 = 0.999
EPS = 1e-15

SPLAT_GROUPS = ("positions", "log_scales", "rotations", "opacity_logits", "colors")

DEFAULT_LRS = {
    "positions": 1.6e-4,
    "log_scales": 5e-3,
    "rotations": 1e-3,
    "opacity_logits": 5e-2,
    "colors": 2.5e-3,
    "pose_rot": 1e-4,
    "pose_trans": 1e-3,
}

POSITION_LR_FINAL_RATIO = 1.6e-6 / 1.6e-4


def position_lr(base: float, iteration: int, max_iter: int) -> float:
    """Exponential decay base -> base * 1e-2 over max_iter (optim.py:33-36)."""
    t = min(max(iteration / max(max_iter, 1), 0.0), 1.0)
    return base * POSITION_LR_FINAL_RATIO ** t


class Adam:
    def __init__(self, lrs: dict | None = None):
        self.lrs = dict(DEFAULT_LRS)
        if lrs:
            self.lrs.update(lrs)
        self._m: dict[str, torch.Tensor] = {}
        self._v: dict[str, torch.Tensor] = {}
        self._steps: dict[str, int] = {}
        self.skipped_rows = 0
        self._skipped_dev = None

    def _state(self, name: str, param: torch.Tensor):
        if name not in self._m:
            self._m[name] = torch.zeros_like(param)
            self._v[name] = torch.zeros_like(param)
            self._steps[name] = 0
        if self._m[name].shape != param.shape:
            raise ValueError(
                f"group {name}: moment shape {tuple(self._m[name].shape)} does not "
                f"match parameter shape {tuple(param.shape)}; resize after densify")
        return self._m[name], self._v[name]

    def _group(self, name, p, g, lr_overrides) -> _lib.AdamGroup_t:
        if not (isinstance(p, torch.Tensor) and p.is_cuda and p.dtype == torch.float32
                and p.is_contiguous()):
            raise TypeError(f"group {name}: parameters must be contiguous FP32 CUDA tensors")
        if p.dim() == 0:
            raise ValueError(f"group {name}: scalar parameters unsupported")
        m, v = self._state(name, p)
        lr = (lr_overrides or {}).get(name, self.lrs.get(name, 1e-3))
        self._steps[name] += 1
        t = self._steps[name]
        rows = p.shape[0]
        width = p.numel() // rows if rows else 1
        d = _lib.AdamGroup_t()
        d.param = p.data_ptr()
        d.grad = g.data_ptr() if g is not None else None
        d.exp_avg = m.data_ptr()
        d.exp_avg_sq = v.data_ptr()
        d.rows = rows
        d.width = width
        d.renormalize = 1 if name == "rotations" else 0
        d.lr = lr
        d.bias_correction1 = 1.0 - BETA1 ** t
        d.bias_correction2 = 1.0 - BETA2 ** t
        return d

    def _counter(self) -> torch.Tensor:
        if self._skipped_dev is None:
            self._skipped_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
        return self._skipped_dev

    def step_async(self, params: dict, grads: dict, lr_overrides=None) -> torch.Tensor:
        """Launch the update; returns the device counter of skipped rows
        (cumulative) without synchronising."""
        lib = _lib.load()
        descs = []
        keep = []
        for name, p in params.items():
            g = grads[name]
            g = g.to(device=p.device, dtype=torch.float32).contiguous() \
                if isinstance(g, torch.Tensor) else torch.as_tensor(
                    np.asarray(g, dtype=np.float32), device=p.device)
            if g.numel() != p.numel():
                raise ValueError(f"group {name}: gradient shape {tuple(g.shape)} does not "
                                 f"match parameter shape {tuple(p.shape)}")
            keep.append(g)
            descs.append(self._group(name, p, g, lr_overrides))
        counter = self._counter()
        for i in range(0, len(descs), _lib.MAX_ADAM_GROUPS):
            chunk = descs[i: i + _lib.MAX_ADAM_GROUPS]
            arr = (_lib.AdamGroup_t * len(chunk))(*chunk)
            _lib.check(lib.tsr_adam_step(arr, len(chunk), counter.data_ptr(),
                                         _lib.stream_handle()), "tsr_adam_step")
        return counter

    def step(self, params: dict, grads: dict, lr_overrides=None) -> int:
        """In-place bias-corrected Adam update; returns skipped row count."""
        before = int(self._counter().item())
        after = int(self.step_async(params, grads, lr_overrides).item())
        skipped = after - before
        self.skipped_rows += skipped
        return skipped

    def groups_for_fused(self, params: dict, lr_overrides=None, advance: bool = True):
        """Descriptors for the fused K4b+K5 kernel (grads come from registers).
        advance=False builds them without counting a step (CUDA-graph capture,
        where lr / bias corrections come from device memory instead)."""
        if not advance:
            steps = dict(self._steps)
        descs = [self._group(name, params[name], None, lr_overrides) for name in SPLAT_GROUPS]
        if not advance:
            self._steps.update(steps)
        return (_lib.AdamGroup_t * 5)(*descs)

    def resize(self, decisions) -> None:
        """Mirror a densify/prune mutation on the moments (optim.py:90-111)."""
        n_old = len(decisions)
        codes = getattr(decisions, "codes", None)
        if codes is not None:  # density.Decisions: device action codes
            from .density import CLONE, PRUNE, SPLIT
            keep = (codes != PRUNE) & (codes != SPLIT)
            n_new = int((codes == CLONE).sum()) + 2 * int((codes == SPLIT).sum())
        else:
            keep = torch.tensor([d.action not in ("prune", "split") for d in decisions],
                                dtype=torch.bool, device="cuda")
            n_new = sum(d.action == "clone" for d in decisions) + \
                2 * sum(d.action == "split" for d in decisions)
        for name in SPLAT_GROUPS:
            if name not in self._m:
                continue
            if self._m[name].shape[0] != n_old:
                raise ValueError(f"group {name}: {self._m[name].shape[0]} moment rows but "
                                 f"{n_old} decisions")
            for store in (self._m, self._v):
                old = store[name]
                zeros = torch.zeros((n_new,) + tuple(old.shape[1:]), device=old.device)
                store[name] = torch.cat([old[keep], zeros]).contiguous()

    def reset_group(self, name: str) -> None:
        if name in self._m:
            self._m[name].zero_()
            self._v[name].zero_()
            self._steps[name] = 0

    def moments(self, name):
        return self._m.get(name), self._v.get(name)
