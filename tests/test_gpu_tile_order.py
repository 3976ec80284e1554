"""Heavy-tile-first launch order (tsr_tile_order, SURVEY §7.3 #4 / north
star (3)): a permutation with the tiles longer than 4x the mean first (raster
order within both classes), and K3 renders bitwise the same buffers in that
order as in raster order (one CTA per tile; the order only moves the heavy
tiles' CTAs to the front of the launch)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_heavy_first_order_is_a_permutation_and_renders_identically():
    import paper_2601_19489_b200 as ts
    from paper_2601_19489_b200 import _lib
    from paper_2601_19489_b200.forward import RenderTargets, render_raw
    from paper_2601_19489_b200.synthetic import make_scene
    params, cam, _ = make_scene(200_000, 640, 480, seed=3, clustered=True,
                                cluster_opacity=(0.005, 0.03))
    gset = ts.GaussianSet(**params)
    camera = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 640, 480, cam["R"], cam["t"])
    vr = ts.render_view(gset, camera, ts.TrainConfig())
    tiles = vr.tiles
    n_tiles = tiles.tiles_x * tiles.tiles_y
    order = torch.empty(n_tiles + 1, dtype=torch.int32, device="cuda")
    lib = _lib.load()
    _lib.check(lib.tsr_tile_order(tiles.offsets.data_ptr(), n_tiles, order.data_ptr(),
                                  _lib.stream_handle()), "tsr_tile_order")
    o = order.cpu().numpy()
    assert o[-1] == 1  # the clustered scene has heavy tiles
    perm = o[:-1]
    assert np.array_equal(np.sort(perm), np.arange(n_tiles))
    lens = np.diff(tiles.offsets.cpu().numpy())
    heavy = lens > max(4 * lens.sum() // n_tiles, 64)
    h = int(heavy.sum())
    assert heavy[perm[:h]].all() and not heavy[perm[h:]].any()
    assert np.all(np.diff(perm[:h]) > 0) and np.all(np.diff(perm[h:]) > 0)
    outs = []
    for od in (None, order):
        t = RenderTargets(480, 640, tiles.n_pairs // 32 + n_tiles + 1)
        render_raw(vr.batch.rec, tiles.values, tiles.offsets, tiles.ckpt_base, 640, 480,
                   np.zeros(3), t, tile_order=od)
        outs.append(t)
    torch.cuda.synchronize()
    for k in ("color", "depth", "final_T", "n_contrib", "n_considered"):
        assert torch.equal(getattr(outs[0], k), getattr(outs[1], k)), k
