"""Region-culled K3 + K4 (render.cu kCkpt 3, backward_regions.cu) -- the
training step's pair -- through the C-ABI, against the oracle
(backward_per_gaussian, backward.py:137-223) and against the per-tile K4.

Bars: the region render's outputs are the reference-checkpoint render's bit
for bit (the culling only skips exact zeros); Grad2D max|x - y| / max|y| <=
1e-4 per field against the oracle (the reference's metric,
test_backward.py:34-39); merges equal the reference's count.  Scenes cover
one segment per tile (C1), many segments per tile (a low-opacity cluster:
pixels alive over several 1024-position segments), the depth and final-T
channels, and frames whose size is not a multiple of the tile; both region
shapes (8x8 regions with 16-lane pipelines, 8x4 with 8-lane ones)."""

import numpy as np
import pytest
import torch

from conftest import host_batch, host_index, np64, rel_err
from oracle import raster as O

pytestmark = pytest.mark.gpu

GRAD_RTOL = 1e-4
FIELDS = ("d_means2d", "d_conics", "d_opacities", "d_colors", "d_depths")


def regions_pass(vr, grad_color, grad_depth=None, grad_final_T=None, background=(0.0, 0.0, 0.0),
                 region_height=None):
    """K3 (region mode) + K4r on a render_view's batch and index."""
    import paper_2601_19489_b200 as ts
    from paper_2601_19489_b200.backward import backward_regions_raw
    from paper_2601_19489_b200.forward import RegionLists, RenderTargets, render_regions_raw
    b, t = vr.batch, vr.tiles
    p = max(t.n_pairs, 1)
    tgt = RenderTargets(b.height, b.width, p // 32 + t.tiles_x * t.tiles_y + 1)
    reg = RegionLists(b.width, b.height, p, region_height)
    render_regions_raw(b.rec, t.values if t.n_pairs else None, t.offsets, t.ckpt_base, b.width,
                       b.height, background, tgt, reg)
    out = torch.zeros((len(b), 10), dtype=torch.float32, device="cuda")
    merges = torch.zeros(1, dtype=torch.int64, device="cuda")
    f32 = lambda a: None if a is None else torch.as_tensor(a, dtype=torch.float32, device="cuda")
    backward_regions_raw(b.rec, t.values if t.n_pairs else None, t.offsets, b.width, b.height,
                         tgt, t.ckpt_base, reg, f32(grad_color), f32(grad_depth),
                         f32(grad_final_T), out, merges)
    torch.cuda.synchronize()
    return tgt, reg, ts.Grad2D(out, int(merges.item()))


def _scene(n, w, h, seed=0, clustered=False, cluster_opacity=None):
    import paper_2601_19489_b200 as ts
    params, cam, gt = O.make_scene(n, w, h, seed=seed, clustered=clustered,
                                   cluster_opacity=cluster_opacity)
    gset = ts.GaussianSet(**params)
    camera = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], w, h, cam["R"], cam["t"])
    vr = ts.render_view(gset, camera, ts.TrainConfig())
    return ts, vr, gt


def _vs_oracle(vr, gcol, gdep=None, gT=None, region_height=None):
    hb, hi = host_batch(vr.batch), host_index(vr.tiles)
    colors = np64(vr.colors)
    ob = O.render(hb, hi, colors, np.zeros(3))
    tgt, reg, g2 = regions_pass(vr, gcol, gdep, gT, region_height=region_height)
    # the region render is the reference-checkpoint render, bit for bit
    for k in ("color", "depth", "final_T", "n_contrib", "n_considered"):
        assert torch.equal(getattr(tgt, k), getattr(vr.buffers, k)), k
    og = O.backward_per_gaussian(ob, hb, hi, colors, gcol, gdep, gT)
    errs = {k: rel_err(np64(getattr(g2, k)), og[k]) for k in FIELDS
            if np.abs(og[k]).max(initial=0.0) > 0}
    for k, e in errs.items():
        assert e < GRAD_RTOL, (k, errs)
    assert g2.merges == og["merges"]
    return tgt, reg, g2, errs


@pytest.mark.parametrize("region_height", [4, 8])
@pytest.mark.parametrize("n,w,h", [(10_000, 256, 256), (3_000, 200, 120), (20_000, 64, 64)])
def test_regions_backward_vs_oracle(n, w, h, region_height):
    ts, vr, gt = _scene(n, w, h)
    assert int(torch.diff(vr.tiles.offsets).max()) > 0
    rng = np.random.default_rng(n)
    gcol = rng.normal(0, 1e-3, (h, w, 3))
    _vs_oracle(vr, gcol, region_height=region_height)


@pytest.mark.parametrize("region_height", [4, 8])
def test_regions_many_segments_per_tile(region_height):
    """A low-opacity cluster (C3-lo style): pixels stay alive for thousands
    of list positions, so their tiles' work spans several segments (units),
    each starting from K3's segment-start checkpoint."""
    ts, vr, gt = _scene(30_000, 64, 64, seed=3, clustered=True, cluster_opacity=(0.004, 0.02))
    assert int(vr.buffers.n_considered.max()) > 3 * 1024, int(vr.buffers.n_considered.max())
    rng = np.random.default_rng(7)
    _vs_oracle(vr, rng.normal(0, 1e-3, (64, 64, 3)), region_height=region_height)


@pytest.mark.parametrize("region_height", [4, 8])
def test_regions_depth_and_final_T_channels(region_height):
    ts, vr, gt = _scene(5_000, 160, 96, seed=5)
    rng = np.random.default_rng(11)
    _vs_oracle(vr, rng.normal(0, 1e-3, (96, 160, 3)), rng.normal(0, 1e-3, (96, 160)),
               rng.normal(0, 1e-3, (96, 160)), region_height=region_height)


@pytest.mark.parametrize("region_height", [4, 8])
def test_regions_zero_upstream_half_tile(region_height):
    """Upstream zero outside a band of rows: row pairs with no upstream are
    skipped (exact zeros) and merges still count every pair of a tile whose
    upstream is not all zero."""
    ts, vr, gt = _scene(8_000, 128, 128, seed=2)
    g = np.zeros((128, 128, 3))
    g[4:6] = 1e-3  # only the top row pair of the first tile row
    _vs_oracle(vr, g, region_height=region_height)


@pytest.mark.parametrize("region_height", [4, 8])
def test_region_lists_cover_every_blend(region_height):
    """Each region list is increasing, within [0, n), pairs every position
    with its batch row, and holds exactly the
    list positions that blend at >= 1 pixel of the region (the backward's
    participation, oracle alphas; positions whose alpha is within 1e-5 of
    the 1/255 threshold at every such pixel may go either way in FP32)."""
    ts, vr, gt = _scene(4_000, 96, 64, seed=9)
    hb, hi = host_batch(vr.batch), host_index(vr.tiles)
    tgt, reg, _ = regions_pass(vr, np.zeros((64, 96, 3)), region_height=region_height)
    nr = 64 // (2 * region_height)
    # entries are (list position, batch row) pairs
    pairs, seg = reg.list.cpu().numpy().reshape(-1, 2), reg.seg.cpu().numpy()
    lst, lrow = pairs[:, 0], pairs[:, 1]
    off = hi["offsets"]
    for tile in range(hi["tiles_x"] * hi["tiles_y"]):
        lo, n = int(off[tile]), int(off[tile + 1] - off[tile])
        if n == 0:
            continue
        nseg = -(-n // 1024)
        ty, tx = divmod(tile, hi["tiles_x"])
        for r in range(nr):
            total = seg[nr * ((lo >> 10) + tile + nseg - 1) + r]
            ent = lst[nr * lo + r * n: nr * lo + r * n + total].astype(np.int64)
            assert np.all(np.diff(ent) > 0) and (total == 0 or (ent[0] >= 0 and ent[-1] < n))
            rows = lrow[nr * lo + r * n: nr * lo + r * n + total].astype(np.int64)
            assert np.array_equal(rows, np.asarray(hi["values"])[lo + ent]), (tile, r)
            x0, y0 = tx * 16 + 8 * (r & 1), ty * 16 + region_height * (r >> 1)
            x1, y1 = min(x0 + 8, 96), min(y0 + region_height, 64)
            if x0 >= 96 or y0 >= 64:
                continue
            gy, gx = np.mgrid[y0:y1, x0:x1]
            px, py = gx.reshape(-1) + 0.5, gy.reshape(-1) + 0.5
            nc = np64(vr.buffers.n_considered)[y0:y1, x0:x1].reshape(-1)
            need, may = [], []
            for k in range(n):
                al = O._alpha(hb, hi["values"][lo + k], px, py)[0]
                if np.any((al >= (1 / 255) * (1 + 1e-5)) & (k < nc)):
                    need.append(k)
                if np.any((al >= (1 / 255) * (1 - 1e-5)) & (k < nc)):
                    may.append(k)
            assert set(need) <= set(ent.tolist()) <= set(may), (tile, r)


def test_train_step_region_k4_matches_tile_k4(monkeypatch):
    """The training step's K3 + K4 with the region-culled form forced on a
    small frame equals the per-tile form: same render outputs bit for bit,
    Grad2D within the FP32 bar (the two merge the same per-(splat, pixel)
    terms in different orders)."""
    import paper_2601_19489_b200 as ts
    from paper_2601_19489_b200 import backward as bw
    params, cam, gt = O.make_scene(20_000, 320, 200, seed=4)
    camera = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 320, 200, cam["R"], cam["t"])
    gt_t = torch.tensor(gt, dtype=torch.float32, device="cuda")
    out = {}
    for form in ("regions", "tiles"):
        monkeypatch.setattr(bw, "K4_FORM", form)
        monkeypatch.setattr(bw, "REGIONS_MIN_PAIRS", 0)
        st = ts.TrainStep(ts.GaussianSet(**params), ts.TrainConfig(max_iters=100), extent=4.0)
        batch = st.forward(camera)
        st.loss_and_backward(batch, camera, gt_t)
        torch.cuda.synchronize()
        assert (st.regions is not None) == (form == "regions")
        out[form] = (st.targets.color.clone(), st.targets.n_considered.clone(),
                     st.grad2d.clone(), int(st.merges.item()))
    assert torch.equal(out["regions"][0], out["tiles"][0])
    assert torch.equal(out["regions"][1], out["tiles"][1])
    g_r, g_t = np64(out["regions"][2]), np64(out["tiles"][2])
    for f, sl in (("mean", slice(0, 2)), ("conic", slice(2, 5)), ("opacity", slice(5, 6)),
                  ("color", slice(6, 9))):
        assert rel_err(g_r[:, sl], g_t[:, sl]) < GRAD_RTOL, f
    assert out["regions"][3] == out["tiles"][3]


def test_streams_filed_once_with_their_lengths():
    """K3 files one K4r stream per (tile, segment, region) with entries --
    plus every tile's (segment 0, region 0) stream, which counts merges --
    under its length's bucket (width 4 below 256 entries); each record holds
    (tile << 16 | segment << 3 | region, list start, list length, first
    entry, entries) consistent with the index and the segment counts."""
    ts, vr, gt = _scene(30_000, 64, 64, seed=3, clustered=True, cluster_opacity=(0.004, 0.02))
    b, t = vr.batch, vr.tiles
    g = np.zeros((64, 64, 3))
    g[:] = 1e-3
    tgt, reg, _ = regions_pass(vr, g, region_height=8)
    nr, nb = 4, 72
    ctl = reg.ctl.cpu().numpy()
    off = t.offsets.cpu().numpy()
    P, tiles = int(off[-1]), len(off) - 1
    cap = 8 * (P // 1024 + tiles + 1)
    units = reg.units.cpu().numpy().view(np.uint32)
    recs = units[nb * cap:].reshape(-1, 8)
    seg = reg.seg.cpu().numpy()

    def bucket(n):
        return n >> 2 if n < 256 else min(64 + ((n - 256) >> 7), nb - 1)

    seen = {}
    for bk in range(nb):
        for sid in units[bk * cap: bk * cap + int(ctl[bk])]:
            code, start, n, e0, ln = (int(v) for v in recs[sid][:5])
            key = (code >> 16, (code >> 3) & 0x1fff, code & 7)
            assert key not in seen, key
            seen[key] = (start, n, e0, ln)
            assert bucket(ln) == bk, (key, ln, bk)
    assert int(ctl[nb + 1]) == len(seen)  # record ids handed out
    expect = set()
    for tile in range(tiles):
        lo, n = int(off[tile]), int(off[tile + 1] - off[tile])
        if n == 0:
            continue
        for s in range(-(-n // 1024)):
            for r in range(nr):
                cur = int(seg[nr * ((lo >> 10) + tile + s) + r])
                prev = int(seg[nr * ((lo >> 10) + tile + s - 1) + r]) if s else 0
                if cur - prev > 0 or (s == 0 and r == 0):
                    expect.add((tile, s, r))
                    assert seen[(tile, s, r)] == (lo, n, prev, cur - prev), (tile, s, r)
    assert set(seen) == expect
