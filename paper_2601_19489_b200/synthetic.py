"""Seeded synthetic scenes (reference: tilesplat/synthetic.py idioms).

`make_scene` is the canonical generator of SURVEY.md §8(d) used for parity
tests and the benchmark configs; pure NumPy (inputs, not the algorithm).
"""

from __future__ import annotations

import numpy as np


def look_at(eye, target, fx, width, height):
    """world->camera (R, t), x right / y down / z forward (synthetic.py:46-60)."""
    eye = np.asarray(eye, float)
    f = np.asarray(target, float) - eye
    f = f / np.linalg.norm(f)
    r = np.cross(f, np.array([0.0, 1.0, 0.0]))
    if np.linalg.norm(r) < 1e-8:
        r = np.cross(f, np.array([1.0, 0.0, 0.0]))
    r = r / np.linalg.norm(r)
    d = np.cross(f, r)
    R = np.stack([r, d, f])
    return dict(fx=fx, fy=fx, cx=width / 2.0, cy=height / 2.0, width=width, height=height,
                R=R, t=-R @ eye)


def ring_poses(n_views, radius, fx, width, height):
    """Pose dicts of a full camera ring looking at the origin (the bench's
    view-parallel cameras; synthetic.py:63-76)."""
    cams = []
    for i in range(n_views):
        phi = 2.0 * np.pi * i / n_views
        eye = np.array([radius * np.sin(phi), 0.0, -radius * np.cos(phi)])
        cams.append(look_at(eye, (0.0, 0.0, 0.0), fx, width, height))
    return cams


def look_at_camera(eye, target, fx, width, height, name=""):
    """A `Camera` at eye looking at target (synthetic.py:46-60)."""
    from .scene import Camera
    p = look_at(eye, target, fx, width, height)
    return Camera(p["fx"], p["fy"], p["cx"], p["cy"], width, height, p["R"], p["t"], name=name)


def camera_ring(n_views: int, radius: float = 4.0, fx: float = 45.0, width: int = 48,
                height: int = 48, z_offset: float = 0.0, arc_degrees: float = 360.0):
    """Cameras on a ring (or an arc of it) looking at the origin
    (synthetic.py:63-76)."""
    cams = []
    full = abs(arc_degrees - 360.0) < 1e-9
    for i in range(n_views):
        span = np.deg2rad(arc_degrees)
        phi = span * i / n_views if full else span * (i / max(n_views - 1, 1) - 0.5)
        eye = np.array([radius * np.sin(phi), z_offset, -radius * np.cos(phi)])
        cams.append(look_at_camera(eye, (0.0, 0.0, 0.0), fx, width, height,
                                   name=f"view_{i:04d}.png"))
    return cams


def random_gaussian_set(n_splats: int, seed: int = 0, spread: float = 0.8,
                        scale_range=(0.12, 0.3), opacity_range=(0.5, 0.9), sh_degree: int = 0):
    """synthetic.py:79-96 (host draw, uploaded once)."""
    from .scene import GaussianSet
    rng = np.random.default_rng(seed)
    colors = np.zeros((n_splats, (sh_degree + 1) ** 2, 3))
    colors[:, 0, :] = rng.uniform(0.15, 0.85, (n_splats, 3))
    if sh_degree > 0:
        colors[:, 1:, :] = rng.normal(0.0, 0.05, colors[:, 1:, :].shape)
    quats = rng.normal(0.0, 1.0, (n_splats, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    op = rng.uniform(*opacity_range, n_splats)
    return GaussianSet(positions=rng.uniform(-spread, spread, (n_splats, 3)),
                       log_scales=np.log(rng.uniform(*scale_range, (n_splats, 3))),
                       rotations=quats, opacity_logits=np.log(op / (1.0 - op)), colors=colors)


def synthetic_scene(n_splats: int = 10, n_views: int = 5, width: int = 48, height: int = 48,
                    seed: int = 0, fx: float = 45.0, with_depth: bool = True,
                    background=(0.0, 0.0, 0.0), arc_degrees: float = 360.0, gt_set=None):
    """Self-consistent scene (synthetic.py:99-122): GT splats rendered by the
    B200 renderer become the ground-truth images (and exact depth priors).
    Returns (scene, gt_set).  `gt_set` overrides the random GT splats (the C5
    workload renders the canonical 1M-splat scene into its views)."""
    import torch
    from .ingest import Scene
    from .trainer import TrainConfig, render_view
    if gt_set is None:
        gt_set = random_gaussian_set(n_splats, seed=seed)
    cams = camera_ring(n_views, fx=fx, width=width, height=height, arc_degrees=arc_degrees)
    cfg = TrainConfig(round_profile="round2", max_iters=1, background=background)
    for cam in cams:
        vr = render_view(gt_set, cam, cfg, checkpoints=False)
        b = vr.buffers
        # ground truth stays resident on the device (FP32), like every image
        cam.gt_image = torch.clamp(b.color, 0.0, 1.0).clone()
        if with_depth:
            cam.depth_prior = b.normalized_depth().clone()
            cam.depth_valid = (b.n_contrib > 0) & (cam.depth_prior > 0)
    h = gt_set.to_numpy()
    scene = Scene(cameras=cams, points=h["positions"].copy(),
                  colors=(np.clip(h["colors"][:, 0, :], 0, 1) * 255).astype(np.uint8),
                  extent=4.0 * 1.1)
    return scene, gt_set


def make_scene(n, width, height, seed=0, clustered=False, sh_degree=0, cluster_opacity=None):
    """Canonical synthetic scene of SURVEY.md §8(d).  Every parameter is made
    FP32-representable so the CPU oracle and the FP32 device see identical
    inputs.  cluster_opacity=(lo, hi) redraws the clustered half's opacities
    from U(lo, hi) -- the low-opacity "C3-lo" stress case of SURVEY §7.3 #4,
    whose cluster tiles need thousands of blends per pixel to terminate (drawn
    after everything else, so the other parameters equal C3's)."""
    rng = np.random.default_rng(seed)
    fx = 1600.0 * width / 1920.0
    pos = rng.uniform(-1.0, 1.0, (n, 3)) * np.array([1.5, 1.5 * height / width, 1.0])
    if clustered:
        k = n - n // 2
        pos[n // 2:] = rng.normal((0.3, 0.1, -0.5), (0.08, 0.08, 0.03), (k, 3))
    log_scales = np.log(rng.uniform(0.002, 0.012, (n, 3)) * (1600.0 / fx))
    q = rng.normal(0.0, 1.0, (n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    op = rng.uniform(0.05, 0.95, n)
    logits = np.log(op / (1.0 - op))
    C = (sh_degree + 1) ** 2
    colors = np.zeros((n, C, 3))
    colors[:, 0, :] = rng.uniform(0.0, 1.0, (n, 3))
    if C > 1:
        colors[:, 1:, :] = rng.normal(0.0, 0.05, (n, C - 1, 3))
    gt = rng.uniform(0.0, 1.0, (height, width, 3))
    if clustered and cluster_opacity is not None:
        lo, hi = cluster_opacity
        oc = rng.uniform(lo, hi, n - n // 2)
        logits[n // 2:] = np.log(oc / (1.0 - oc))
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    params = dict(positions=f32(pos), log_scales=f32(log_scales), rotations=f32(q),
                  opacity_logits=f32(logits), colors=f32(colors))
    cam = look_at((0.0, 0.0, -4.0), (0.0, 0.0, 0.0), fx, width, height)
    return params, cam, f32(gt)


def random_splat_batch(n_splats: int, anisotropy: float = 1.0, seed: int = 0, width: int = 640,
                       height: int = 480, sigma_range=(0.8, 4.0)):
    """Random PD conics at a given anisotropy (synthetic.py:16-43), drawn on
    the host in float64 exactly as the reference draws them, then stored as
    the device batch (FP32)."""
    from .projection import SplatBatch
    rng = np.random.default_rng(seed)
    means = np.stack([rng.uniform(0, width, n_splats), rng.uniform(0, height, n_splats)], axis=1)
    minor = rng.uniform(*sigma_range, n_splats)
    major = minor * anisotropy
    theta = rng.uniform(0.0, np.pi, n_splats)
    ct, st = np.cos(theta), np.sin(theta)
    inv1, inv2 = 1.0 / major ** 2, 1.0 / minor ** 2
    a = ct * ct * inv1 + st * st * inv2
    c = st * st * inv1 + ct * ct * inv2
    b = ct * st * (inv1 - inv2)
    opacities = rng.uniform(0.05, 0.98, n_splats)
    return SplatBatch(means, np.stack([a, b, c], axis=1),
                      np.maximum(0.0, 2.0 * np.log(255.0 * opacities)),
                      rng.uniform(0.1, 20.0, n_splats), opacities,
                      np.arange(n_splats, dtype=np.int64), width, height)
