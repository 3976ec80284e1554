"""Generate golden vectors from the UNMODIFIED reference (tilesplat).

Run in the build container (it imports /root/reference/pkg/src, which does
not exist on the GPU box):

    python tests/golden/make_golden.py

Every input is rounded to FP32 first, so the device (FP32 storage) sees
bit-identical inputs and binning outputs must match these files exactly.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(OUT.parents[1]))

from tilesplat import binning, losses, optim, synthetic  # noqa: E402
from tilesplat.backward import backward_per_gaussian, backward_per_pixel  # noqa: E402
from tilesplat.forward import render  # noqa: E402
from tilesplat.projection import SplatBatch, project, project_vjp  # noqa: E402
from tilesplat.scene import Camera, GaussianSet  # noqa: E402

from oracle.raster import make_scene  # noqa: E402


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def batch_arrays(b, prefix=""):
    return {prefix + "means2d": b.means2d, prefix + "conics": b.conics,
            prefix + "level_t": b.level_t, prefix + "depths": b.depths,
            prefix + "opacities": b.opacities, prefix + "source_ids": b.source_ids,
            prefix + "wh": np.array([b.width, b.height])}


def f32_batch(b):
    return SplatBatch(f32(b.means2d), f32(b.conics), f32(b.level_t), f32(b.depths),
                      f32(b.opacities), b.source_ids.copy(), b.width, b.height)


def index_arrays(idx, prefix):
    return {prefix + "keys": idx.keys, prefix + "values": idx.values,
            prefix + "offsets": idx.offsets,
            prefix + "checksum": np.array(idx.checksum())}


def golden_binning():
    out = {}
    cases = [
        ("rand", synthetic.random_splat_batch(500, anisotropy=8.0, seed=3)),
        ("aniso", synthetic.random_splat_batch(2000, anisotropy=15.0, seed=11, width=640,
                                               height=480, sigma_range=(0.5, 2.5))),
        ("small", synthetic.random_splat_batch(40, anisotropy=5.0, seed=7, width=160,
                                               height=160, sigma_range=(0.3, 3.0))),
    ]
    # pinned edge cases (test_binning.py:152-164, 105-108, 50-54)
    tang = SplatBatch(np.array([[30.0, 30.0], [30.0, 30.0], [40.0, 40.0], [-50.0, -50.0],
                                [24.0, 24.0], [25.0, 25.0]]),
                      np.array([[1.0, 0.0, 1.0]] * 6), np.array([4.0, 8.0, 0.0, 4.0, 1.0, 1.0]),
                      np.array([1.0, 1.5, 2.0, 1.0, 2.0, 2.0]),
                      np.exp(np.array([4.0, 8.0, 0.0, 4.0, 1.0, 1.0]) / 2.0) / 255.0,
                      np.arange(6), 128, 128)
    cases.append(("edge", tang))
    for name, b in cases:
        b = f32_batch(b)
        binning.compute_snugboxes(b)
        out.update(batch_arrays(b, name + "_"))
        out[name + "_rect"] = b.tile_rect
        out[name + "_xmin"] = b.x_min
        out[name + "_ymax"] = b.y_max
        seq = binning.bin_sequential(b)
        lb = binning.bin_load_balanced(b)
        assert seq.checksum() == lb.checksum()
        out.update(index_arrays(seq, name + "_seq_"))
    np.savez_compressed(OUT / "binning.npz", **out)


def raster_scene(rng, n, width, height, opacity_range=(0.1, 0.85), sigma_range=(3.0, 9.0)):
    """Random 2D scene in the style of test_backward.random_scene."""
    sig = rng.uniform(*sigma_range, n)
    ops = rng.uniform(*opacity_range, n)
    conics = np.stack([1 / sig ** 2, rng.uniform(-0.4, 0.4, n) / sig ** 2, 1 / sig ** 2], 1)
    means = np.stack([rng.uniform(0, width, n), rng.uniform(0, height, n)], 1)
    b = SplatBatch(f32(means), f32(conics), f32(np.maximum(0.0, 2 * np.log(255 * ops))),
                   f32(rng.uniform(1, 6, n)), f32(ops), np.arange(n), width, height)
    return b, f32(rng.uniform(0, 1, (n, 3)))


def golden_raster():
    out = {}
    rng = np.random.default_rng(2024)
    specs = [("r60", 60, 32, 32, (0.1, 0.85), (3.0, 9.0)),
             ("r128", 128, 40, 24, (0.1, 0.85), (3.0, 9.0)),
             ("deep", 100, 16, 16, (0.02, 0.12), (8.0, 16.0)),
             ("opaque", 64, 16, 16, (0.85, 0.95), (10.0, 16.0))]
    for name, n, w, h, orng, srng in specs:
        b, colors = raster_scene(rng, n, w, h, orng, srng)
        tiles = binning.bin_sequential(b)
        bg = np.array([0.2, 0.1, 0.3])
        bufs = render(b, tiles, colors, bg)
        g_c = f32(rng.normal(0, 1, (h, w, 3)))
        g_d = f32(rng.normal(0, 1, (h, w)))
        g_t = f32(rng.normal(0, 1, (h, w)))
        gg = backward_per_gaussian(bufs, b, tiles, colors, g_c, g_d, g_t)
        gp = backward_per_pixel(bufs, b, tiles, colors, g_c, g_d, g_t)
        out.update(batch_arrays(b, name + "_"))
        out.update(index_arrays(tiles, name + "_"))
        out[name + "_colors"] = colors
        out[name + "_bg"] = bg
        for k in ("color", "depth", "final_T", "n_contrib", "n_considered"):
            out[f"{name}_{k}"] = getattr(bufs, k)
        for t, ck in bufs.checkpoints.items():
            out[f"{name}_ckpt_{t}"] = ck
        out[name + "_gc"], out[name + "_gd"], out[name + "_gt"] = g_c, g_d, g_t
        for k in ("d_means2d", "d_conics", "d_opacities", "d_colors", "d_depths"):
            out[f"{name}_pg_{k}"] = getattr(gg, k)
            out[f"{name}_pp_{k}"] = getattr(gp, k)
        out[name + "_merges"] = np.array(gg.merges)
    np.savez_compressed(OUT / "raster.npz", **out)


def golden_scene():
    """End-to-end small scene with the canonical generator."""
    out = {}
    for name, n, w, h, clustered, deg in (("s0", 3000, 128, 96, False, 0),
                                          ("s1", 2000, 96, 64, True, 0),
                                          ("sh", 500, 64, 48, False, 2)):
        params, cam, gt = make_scene(n, w, h, seed=5, clustered=clustered, sh_degree=deg)
        gset = GaussianSet(**params)
        camera = Camera(fx=cam["fx"], fy=cam["fy"], cx=cam["cx"], cy=cam["cy"], width=w,
                        height=h, rotation=cam["R"], translation=cam["t"])
        batch = project(gset, camera, near=0.01)
        out.update({f"{name}_p_{k}": v for k, v in params.items()})
        out[f"{name}_cam_R"], out[f"{name}_cam_t"] = cam["R"], cam["t"]
        out[f"{name}_cam_f"] = np.array([cam["fx"], cam["fy"], cam["cx"], cam["cy"], w, h])
        out[f"{name}_gt"] = gt
        out.update(batch_arrays(batch, name + "_b_"))
        from tilesplat.trainer import _splat_colors
        colors, _ = _splat_colors(gset, batch, camera, None)
        out[f"{name}_colors"] = colors
        # raster on the FP32-rounded batch (what the device stores)
        b32 = f32_batch(batch)
        c32 = f32(colors)
        tiles = binning.bin_sequential(b32)
        bufs = render(b32, tiles, c32, np.zeros(3))
        rep, gcol = losses.photometric(bufs.color, gt, 0.2)
        g2 = backward_per_gaussian(bufs, b32, tiles, c32, gcol)
        out.update(index_arrays(tiles, name + "_"))
        for k in ("color", "depth", "final_T", "n_contrib", "n_considered"):
            out[f"{name}_{k}"] = getattr(bufs, k)
        out[f"{name}_loss"] = np.array([rep.photometric, rep.l1, rep.ssim])
        out[f"{name}_gcol"] = gcol
        for k in ("d_means2d", "d_conics", "d_opacities", "d_colors", "d_depths"):
            out[f"{name}_g2_{k}"] = getattr(g2, k)
        g3, gpose = project_vjp(gset, camera, batch, g2, near=0.01)
        for k in ("positions", "log_scales", "rotations", "opacity_logits"):
            out[f"{name}_g3_{k}"] = getattr(g3, k)
        out[f"{name}_pose"] = np.concatenate([gpose.rot_vec, gpose.trans])
    np.savez_compressed(OUT / "scene.npz", **out)


def golden_adam():
    out = {}
    rng = np.random.default_rng(9)
    opt = optim.Adam({"positions": 1e-2, "rotations": 0.1, "colors": 3e-3})
    p = {"positions": f32(rng.normal(0, 1, (7, 3))),
         "rotations": f32(rng.normal(0, 1, (7, 4))),
         "colors": f32(rng.normal(0, 1, (7, 4, 3)))}
    for k, v in p.items():
        out[f"init_{k}"] = v.copy()
    for step in range(4):
        g = {k: f32(rng.normal(0, 1, v.shape)) for k, v in p.items()}
        if step == 1:
            g["positions"][2, 1] = np.nan
            g["colors"][5, 3, 0] = np.inf
        if step == 2:
            g["rotations"][:] *= 1e-20  # tiny-gradient case
        for k, v in g.items():
            out[f"g{step}_{k}"] = v
        out[f"skipped{step}"] = np.array(opt.step(p, g))
        for k, v in p.items():
            out[f"p{step}_{k}"] = v.copy()
            out[f"m{step}_{k}"] = opt.moments(k)[0].copy()
            out[f"v{step}_{k}"] = opt.moments(k)[1].copy()
    np.savez_compressed(OUT / "adam.npz", **out)


def golden_loss():
    rng = np.random.default_rng(4)
    r = f32(rng.uniform(0, 1, (40, 56, 3)))
    g = f32(rng.uniform(0, 1, (40, 56, 3)))
    rep, grad = losses.photometric(r, g, 0.2)
    np.savez_compressed(OUT / "loss.npz", rendered=r, gt=g,
                        values=np.array([rep.photometric, rep.l1, rep.ssim]), grad=grad)


def golden_projection():
    """project / project_vjp on the test_projection.py-style random set."""
    rng = np.random.default_rng(1234)
    n = 40
    params = dict(positions=f32(rng.normal(0, 0.3, (n, 3)) + [0, 0, 3.0]),
                  log_scales=f32(np.log(rng.uniform(0.8, 1.4, (n, 3)) * 0.05)),
                  rotations=f32(rng.normal(0, 1, (n, 4))),
                  opacity_logits=f32(rng.uniform(-2, 2, n)),
                  colors=f32(rng.uniform(0.2, 0.8, (n, 1, 3))))
    params["opacity_logits"][3] = -7.0  # culled (o < 1/255)
    params["positions"][5] = [0.0, 0.0, -1.0]  # behind the camera
    gset = GaussianSet(**params)
    from tilesplat.pose import rodrigues
    R = rodrigues([0.05, -0.1, 0.02])
    cam = Camera(fx=55.0, fy=50.0, cx=32.0, cy=32.0, width=64, height=64, rotation=R,
                 translation=np.array([0.02, -0.03, 0.1]))
    batch = project(gset, cam, near=0.1)
    m = len(batch)

    class G:
        pass

    g2 = G()
    g2.d_means2d = f32(rng.normal(0, 1, (m, 2)))
    g2.d_conics = f32(rng.normal(0, 1, (m, 3)))
    g2.d_depths = f32(rng.normal(0, 1, m))
    g2.d_opacities = f32(rng.normal(0, 1, m))
    g3, gpose = project_vjp(gset, cam, batch, g2, near=0.1)
    out = {f"p_{k}": v for k, v in params.items()}
    out.update(cam_R=cam.rotation, cam_t=cam.translation, cam_f=np.array([55.0, 50.0, 32.0,
                                                                           32.0, 64, 64]))
    out.update(batch_arrays(batch, "b_"))
    out.update(g_means=g2.d_means2d, g_conics=g2.d_conics, g_depths=g2.d_depths,
               g_opac=g2.d_opacities)
    for k in ("positions", "log_scales", "rotations", "opacity_logits"):
        out[f"g3_{k}"] = getattr(g3, k)
    out["pose"] = np.concatenate([gpose.rot_vec, gpose.trans])
    np.savez_compressed(OUT / "projection.npz", **out)


def golden_density():
    """Scoring render, error masks, scores, decisions and moment resize
    (density.py, forward.py:132-137, optim.py:90-111)."""
    from tilesplat import density
    from tilesplat.optim import Adam
    out = {}
    rng = np.random.default_rng(77)
    masks, pix, ids, e_ph = [], [], [], []
    for v, (n, w, h) in enumerate(((90, 48, 40), (90, 48, 40))):
        b, colors = raster_scene(rng, n, w, h, (0.1, 0.85), (2.0, 7.0))
        tiles = binning.bin_sequential(b)
        bufs, con = render(b, tiles, colors, np.zeros(3), scoring=True)
        gt = f32(rng.uniform(0, 1, (h, w, 3)))
        rep, _ = losses.photometric(bufs.color, gt, 0.2)
        m = density.error_mask(bufs.color, gt, 0.5)
        out.update(batch_arrays(b, f"v{v}_"))
        out[f"v{v}_colors"] = colors
        out[f"v{v}_gt"] = gt
        out[f"v{v}_color"] = bufs.color
        out[f"v{v}_pix"] = con.pixel_idx
        out[f"v{v}_rows"] = con.splat_rows
        out[f"v{v}_mask"] = m.mask
        out[f"v{v}_e"] = m.e
        out[f"v{v}_ephoto"] = np.array(rep.photometric)
        masks.append(m)
        pix.append(con.pixel_idx)
        ids.append(b.source_ids[con.splat_rows])
        e_ph.append(rep.photometric)
    out["s_plus"] = density.score_densify(masks, pix, ids, 90)
    out["s_minus"] = density.score_prune(masks, pix, ids, e_ph, 90)
    # decisions on a small 3D set with chosen scores (all four actions + floor guard)
    params, _, _ = make_scene(200, 64, 48, seed=9)
    gset = GaussianSet(**params)
    sp = f32(rng.uniform(0, 30, 200))
    sm = f32(rng.uniform(0, 1, 200))
    for name, min_splats in (("dec", 16), ("floor", 190)):
        new, dec = density.apply_decisions(gset, sp, sm, 16.0, 0.9, 0.01,
                                           np.random.default_rng(5), min_splats=min_splats)
        for k in ("positions", "log_scales", "rotations", "opacity_logits", "colors"):
            out[f"{name}_new_{k}"] = getattr(new, k)
        out[f"{name}_actions"] = np.array(
            [["keep", "clone", "split", "prune"].index(d.action) for d in dec])
        if name == "dec":
            opt = Adam()
            p = {k: getattr(gset, k).copy() for k in ("positions", "log_scales", "rotations",
                                                         "opacity_logits", "colors")}
            g = {k: f32(rng.normal(0, 1, v.shape)) for k, v in p.items()}
            opt.step(p, g)
            out["adam_m_before"] = opt.moments("positions")[0].copy()
            opt.resize(dec)
            out["adam_m_after"] = opt.moments("positions")[0].copy()
            out["adam_v_after"] = opt.moments("log_scales")[1].copy()
            out["adam_g_pos"] = g["positions"]
            out["adam_g_ls"] = g["log_scales"]
    out.update({f"set_{k}": v for k, v in params.items()})
    out["dec_sp"], out["dec_sm"] = sp, sm
    np.savez_compressed(OUT / "density.npz", **out)


def golden_ply():
    """A reference-written PLY (SH degree 1) for the drop-in file-format test."""
    from tilesplat.ingest import write_ply
    params, _, _ = make_scene(37, 64, 48, seed=4, sh_degree=1)
    write_ply(GaussianSet(**params), OUT / "ref_sh1.ply")
    np.savez_compressed(OUT / "ply.npz", **params)


def golden_benchtiling():
    """The reference's bench-tiling harness (cli.py:170-183): pairs and
    checksums per strategy for a few (n, anisotropy, seed)."""
    from tilesplat.cli import run_bench_tiling
    out = {}
    for i, (n, an, seed, w, h) in enumerate(((20000, 8.0, 0, 640, 480), (5000, 1.0, 3, 640, 480),
                                             (30000, 15.0, 7, 1280, 720))):
        res = run_bench_tiling(n, an, seed, w, h)
        out[f"c{i}_args"] = np.array([n, an, seed, w, h], dtype=np.float64)
        for r in res:
            out[f"c{i}_{r.strategy}_pairs"] = np.array(r.pairs)
            out[f"c{i}_{r.strategy}_checksum"] = np.array(r.checksum)
        # the same harness on the FP32-rounded batch (what the device stores)
        b = f32_batch(synthetic.random_splat_batch(n, an, seed, width=w, height=h))
        binning.compute_snugboxes(b)
        for name, fn in (("aabb", binning.bin_aabb), ("snug_seq", binning.bin_sequential),
                         ("snug_lb", binning.bin_load_balanced)):
            idx = fn(b)
            out[f"c{i}_f32_{name}_pairs"] = np.array(idx.n_pairs)
            out[f"c{i}_f32_{name}_checksum"] = np.array(idx.checksum())
    np.savez_compressed(OUT / "benchtiling.npz", **out)


def golden_e2e():
    """Acceptance criterion 5 (test_acceptance.py:161-247): the 5-splat 32x32
    scene with a pose delta, photometric + disparity loss; the reference's
    analytic gradients of every parameter class (incl. the pose) and their
    float64 central finite differences (h = 1e-4), on FP32-rounded inputs."""
    from tilesplat import pose as rpose
    from tilesplat.scene import inverse_sigmoid
    from tilesplat.trainer import TrainConfig as RefConfig
    from tilesplat.trainer import _full_grads, render_view, view_loss_and_grads
    rng = np.random.default_rng(3)
    n = 5
    params = dict(positions=f32(rng.normal(0, 0.3, (n, 3)) + [0, 0, 3.0]),
                  log_scales=f32(np.log(rng.uniform(0.8, 1.4, (n, 3)))),
                  rotations=f32(rng.normal(0, 1, (n, 4))),
                  opacity_logits=f32(inverse_sigmoid(rng.uniform(0.3, 0.6, n))),
                  colors=f32(rng.uniform(0.2, 0.8, (n, 1, 3))))
    R = f32(rpose.rodrigues([0.05, -0.1, 0.02]))
    t = f32([0.02, -0.03, 0.1])
    gt = f32(rng.uniform(0, 1, (32, 32, 3)))
    prior = f32(np.full((32, 32), 3.0))
    rot, trans = f32([0.01, -0.02, 0.015]), f32([0.005, 0.01, -0.02])
    bg = f32([0.1, 0.2, 0.3])
    cfg = RefConfig(round_profile="round2", near=0.1, background=tuple(bg))

    def loss_and_grads(ps, rv, tv, want_grads):
        gset = GaussianSet(**{k: v.copy() for k, v in ps.items()})
        cam = Camera(fx=30.0, fy=32.0, cx=16.0, cy=16.0, width=32, height=32, rotation=R,
                     translation=t, gt_image=gt, depth_prior=prior)
        delta = rpose.PoseDelta(rv.copy(), tv.copy())
        vr = render_view(gset, cam, cfg, delta)
        rep, g2 = view_loss_and_grads(cam, cfg, vr, 0.1)
        if not want_grads:
            return rep.total
        return rep.total, _full_grads(gset, cam, cfg, delta, vr, g2)

    total, grads = loss_and_grads(params, rot, trans, True)
    h = 1e-4
    out = {f"p_{k}": v for k, v in params.items()}
    out.update(cam_R=R, cam_t=t, gt=gt, prior=prior, pose_rot=rot, pose_trans=trans, bg=bg,
               total=np.array(total))
    for k, v in grads.items():
        out[f"g_{k}"] = np.asarray(v)

    def fd(get, put):
        base = get().copy()
        g = np.zeros_like(base)
        for i in range(base.size):
            x = base.copy().reshape(-1)
            x[i] += h
            put(x.reshape(base.shape))
            fp = loss_and_grads(params, rot, trans, False)
            x[i] -= 2 * h
            put(x.reshape(base.shape))
            fm = loss_and_grads(params, rot, trans, False)
            put(base)
            g.reshape(-1)[i] = (fp - fm) / (2 * h)
        return g

    for k in list(params):
        out[f"fd_{k}"] = fd(lambda k=k: params[k], lambda x, k=k: params.__setitem__(k, x))
    out["fd_pose_rot"] = fd(lambda: rot, lambda x: rot.__setitem__(slice(None), x))
    out["fd_pose_trans"] = fd(lambda: trans, lambda x: trans.__setitem__(slice(None), x))
    np.savez_compressed(OUT / "e2e.npz", **out)


if __name__ == "__main__":
    golden_e2e()
    golden_benchtiling()
    golden_density()
    golden_ply()
    golden_binning()
    golden_raster()
    golden_scene()
    golden_adam()
    golden_loss()
    golden_projection()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
