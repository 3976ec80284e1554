"""Shared fixtures.  `-m "not gpu"` runs here (no GPU): the oracle against the
reference's golden vectors, host logic, the C-ABI symbol table and the
multi-process (gloo) view-parallel logic.  `-m gpu` tests are the parity
tests proper: CUDA path (through the C-ABI) vs oracle / golden vectors."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")


def golden(name):
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def batch_from(g, prefix):
    """Golden batch arrays -> oracle batch dict."""
    w, h = (int(v) for v in g[prefix + "wh"])
    return dict(means2d=g[prefix + "means2d"], conics=g[prefix + "conics"],
                level_t=g[prefix + "level_t"], depths=g[prefix + "depths"],
                opacities=g[prefix + "opacities"], source_ids=g[prefix + "source_ids"],
                width=w, height=h)


def rel_err(got, ref, floor=1e-12):
    """max |got - ref| / max |ref| -- the reference's gradient metric
    (test_backward.py:34-39)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.abs(got - ref).max(initial=0.0) / max(np.abs(ref).max(initial=0.0), floor))


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def np64(t):
    """device tensor -> float64 / int64 numpy."""
    a = t.detach().cpu().numpy()
    return a.astype(np.float64) if a.dtype.kind == "f" else a.astype(np.int64)


def dev_batch(b):
    """oracle batch dict -> device SplatBatch (FP32; inputs are FP32-exact)."""
    import paper_2601_19489_b200 as ts
    return ts.SplatBatch(b["means2d"], b["conics"], b["level_t"], b["depths"], b["opacities"],
                         b["source_ids"], b["width"], b["height"])


def host_batch(db):
    """device SplatBatch -> oracle batch dict (FP32 values upcast to FP64)."""
    return dict(means2d=np64(db.means2d), conics=np64(db.conics), level_t=np64(db.level_t),
                depths=np64(db.depths), opacities=np64(db.opacities),
                source_ids=np64(db.source_ids), width=db.width, height=db.height)


def host_index(idx):
    return dict(keys=idx.keys.cpu().numpy().astype(np.uint64),
                values=idx.values.cpu().numpy().astype(np.int64),
                offsets=idx.offsets.cpu().numpy().astype(np.int64),
                tiles_x=idx.tiles_x, tiles_y=idx.tiles_y)


def random_splats(n, seed, width, height, anisotropy=(1.0, 20.0), minor=(0.5, 3.0)):
    """FP32-exact random batch (the style of synthetic.random_splat_batch /
    test_acceptance.anisotropic_batch)."""
    rng = np.random.default_rng(seed)
    an = rng.uniform(*anisotropy, n)
    mi = rng.uniform(*minor, n)
    ma = mi * an
    th = rng.uniform(0, np.pi, n)
    ct, st = np.cos(th), np.sin(th)
    i1, i2 = 1 / ma ** 2, 1 / mi ** 2
    op = rng.uniform(0.05, 0.98, n)
    f = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    return dict(means2d=f(np.stack([rng.uniform(-20, width + 20, n),
                                    rng.uniform(-20, height + 20, n)], 1)),
                conics=f(np.stack([ct * ct * i1 + st * st * i2, ct * st * (i1 - i2),
                                   st * st * i1 + ct * ct * i2], 1)),
                level_t=f(np.maximum(0.0, 2 * np.log(255 * op))),
                depths=f(rng.uniform(0.1, 10.0, n)), opacities=f(op),
                source_ids=np.arange(n), width=width, height=height)
