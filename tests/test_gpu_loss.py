"""Fused photometric loss kernel (csrc/loss.cu) vs the reference's golden
vectors and the oracle at 1080p.  FP32 tolerances: loss values 1e-6 absolute,
gradient max-abs error normalised by max |grad| below 1e-4."""

import numpy as np
import pytest
import torch

from conftest import golden, np64, rel_err
from oracle import raster as O

pytestmark = pytest.mark.gpu


def test_loss_matches_reference_golden():
    import paper_2601_19489_b200 as ts
    g = golden("loss")
    rep, grad = ts.photometric(g["rendered"], g["gt"], 0.2)
    assert np.allclose([rep.photometric, rep.l1, rep.ssim], g["values"], atol=1e-6, rtol=0)
    assert rel_err(np64(grad), g["grad"]) < 1e-4


@pytest.mark.parametrize("shape", [(1080, 1920), (37, 53), (5, 7)])
def test_loss_matches_oracle(shape):
    import paper_2601_19489_b200 as ts
    rng = np.random.default_rng(shape[0])
    r = np.asarray(rng.uniform(0, 1, shape + (3,)), np.float32).astype(np.float64)
    gt = np.asarray(rng.uniform(0, 1, shape + (3,)), np.float32).astype(np.float64)
    e, l1, ssim, gref = O.photometric(r, gt, 0.2)
    rep, grad = ts.photometric(r, gt, 0.2)
    assert abs(rep.photometric - e) < 2e-6 and abs(rep.l1 - l1) < 2e-6
    assert abs(rep.ssim - ssim) < 2e-6
    assert rel_err(np64(grad), gref) < 1e-4


def test_loss_rejects_bad_inputs():
    import paper_2601_19489_b200 as ts
    with pytest.raises(ValueError):
        ts.photometric(np.zeros((4, 4, 3)), np.zeros((4, 5, 3)))
    with pytest.raises(ValueError):
        ts.photometric(np.zeros((4, 4, 3)), np.zeros((4, 4, 3)), lam=1.5)
