"""Adam contract of the reference's tests/test_optim.py through K5 on the
device: zero gradients, first step = -lr, NaN rows skipped/counted with
their moments untouched, quaternion renormalisation, moment resizing for
clone/prune/split and its errors, group reset, bitwise determinism, the
position learning-rate schedule."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _t(a):
    import torch
    return torch.as_tensor(np.asarray(a, np.float32), device="cuda").contiguous()


def _decisions(actions):
    from paper_2601_19489_b200.density import DensifyDecision
    return [DensifyDecision(i, a, 0.0, 0.0) for i, a in enumerate(actions)]


def test_zero_grads_leave_params_unchanged():
    from paper_2601_19489_b200.optim import Adam
    p = _t(np.arange(12).reshape(4, 3))
    before = p.clone()
    Adam({"positions": 1e-2}).step({"positions": p}, {"positions": _t(np.zeros((4, 3)))})
    assert bool((p == before).all())


def test_nan_rows_skipped_and_counted():
    from paper_2601_19489_b200.optim import Adam
    opt = Adam({"positions": 1e-2})
    p = _t(np.ones((3, 3)))
    g = np.ones((3, 3))
    g[1, 2] = np.nan
    assert opt.step({"positions": p}, {"positions": _t(g)}) == 1 and opt.skipped_rows == 1
    h = p.cpu().numpy()
    assert np.array_equal(h[1], np.ones(3)) and np.all(h[[0, 2]] < 1.0)
    m, _ = opt.moments("positions")
    assert not bool(m[1].any())


def test_quaternions_renormalized_after_step():
    from paper_2601_19489_b200.optim import Adam
    rng = np.random.default_rng(0)
    q = rng.normal(0, 1, (5, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    qt = _t(q)
    Adam({"rotations": 0.1}).step({"rotations": qt}, {"rotations": _t(rng.normal(0, 1, (5, 4)))})
    assert np.allclose(np.linalg.norm(qt.cpu().numpy(), axis=1), 1.0, atol=1e-6)


def test_resize_clone_prune_split():
    from paper_2601_19489_b200.optim import Adam
    opt = Adam()
    opt.step({"positions": _t(np.ones((3, 3)))}, {"positions": _t(np.arange(9).reshape(3, 3))})
    m0 = opt.moments("positions")[0].cpu().numpy().copy()
    opt.resize(_decisions(["keep"] * 3))
    assert np.array_equal(opt.moments("positions")[0].cpu().numpy(), m0)
    opt.resize(_decisions(["keep", "clone", "keep"]))
    m, v = (t.cpu().numpy() for t in opt.moments("positions"))
    assert m.shape == (4, 3) and not m[3].any() and not v[3].any()
    assert np.array_equal(m[:3], m0)
    m1 = m.copy()  # rows: m0[0], m0[1], m0[2], clone zeros
    opt.resize(_decisions(["keep", "prune", "split", "keep"]))
    m = opt.moments("positions")[0].cpu().numpy()
    assert m.shape == (4, 3)  # 4 - prune - split parent + 2 children
    assert np.array_equal(m[:2], m1[[0, 3]]) and not m[2:].any()


def test_resize_errors():
    from paper_2601_19489_b200.optim import Adam
    opt = Adam()
    opt.step({"positions": _t(np.ones((3, 3)))}, {"positions": _t(np.ones((3, 3)))})
    with pytest.raises(ValueError, match="moment rows"):
        opt.resize(_decisions(["keep"] * 5))
    with pytest.raises(ValueError, match="resize"):
        opt.step({"positions": _t(np.ones((4, 3)))}, {"positions": _t(np.ones((4, 3)))})


def test_reset_group_and_bitwise_determinism():
    from paper_2601_19489_b200.optim import Adam
    opt = Adam()
    opt.step({"colors": _t(np.ones((2, 1, 3)))}, {"colors": _t(np.ones((2, 1, 3)))})
    opt.reset_group("colors")
    m, v = opt.moments("colors")
    assert not bool(m.any()) and not bool(v.any())

    def run():
        o = Adam({"positions": 1e-2})
        rng = np.random.default_rng(9)
        p = _t(rng.normal(0, 1, (6, 3)))
        for _ in range(50):
            o.step({"positions": p}, {"positions": _t(rng.normal(0, 1, (6, 3)))})
        return p.cpu().numpy()

    assert np.array_equal(run(), run())


def test_position_lr_schedule():
    from paper_2601_19489_b200.optim import position_lr
    base = 1.6e-4
    assert position_lr(base, 0, 1000) == pytest.approx(base)
    assert position_lr(base, 1000, 1000) == pytest.approx(base * 1e-2)
    assert position_lr(base, 500, 1000) == pytest.approx(base * 1e-1)
