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


def camera_ring(n_views, radius, fx, width, height):
    """Cameras on a full ring looking at the origin (synthetic.py:63-76)."""
    cams = []
    for i in range(n_views):
        phi = 2.0 * np.pi * i / n_views
        eye = np.array([radius * np.sin(phi), 0.0, -radius * np.cos(phi)])
        cams.append(look_at(eye, (0.0, 0.0, 0.0), fx, width, height))
    return cams


def make_scene(n, width, height, seed=0, clustered=False, sh_degree=0):
    """Canonical synthetic scene of SURVEY.md §8(d).  Every parameter is made
    FP32-representable so the CPU oracle and the FP32 device see identical
    inputs."""
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
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    params = dict(positions=f32(pos), log_scales=f32(log_scales), rotations=f32(q),
                  opacity_logits=f32(logits), colors=f32(colors))
    cam = look_at((0.0, 0.0, -4.0), (0.0, 0.0, 0.0), fx, width, height)
    return params, cam, f32(gt)
