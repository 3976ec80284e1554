"""CPU oracle of the raster path -- TEST INFRASTRUCTURE ONLY (see __init__).

float64 NumPy.  Each function restates the reference algorithm it cites; the
tile-decision arithmetic keeps NumPy's evaluation order of the reference so
(tile, splat) pairs are bit-identical; the sort is expressed as one lexsort
on (key, emission row), which is the order the reference's stable LSD radix
sort over splat-major emission produces (binning.py:142-158).

A batch is a dict with the SplatBatch fields of projection.py:30-54:
means2d (M,2), conics (M,3), level_t, depths, opacities (M,), source_ids,
width, height.  An index is a dict keys (P,) u64, values (P,) i64,
offsets (T+1,) i64, tiles_x, tiles_y.
"""

from __future__ import annotations

import hashlib

import numpy as np
from scipy.ndimage import correlate1d

TILE = 16
COV_DILATION = 0.3          # projection.py:26
MIN_OPACITY = 1.0 / 255.0   # projection.py:27
ALPHA_CAP = 0.99            # forward.py:25
T_TERMINATE = 1e-4          # forward.py:27
GROUP = 32                  # forward.py:28


# ------------------------------------------------------------------ scene --
# Inputs come from the canonical generator (input generation, not the
# algorithm under test), shared with bench.py's device arm.
from paper_2601_19489_b200.synthetic import camera_ring, look_at, make_scene  # noqa: E402,F401


def _rotmat(q):
    """quaternion (w,x,y,z), normalised inside (scene.py:33-47)."""
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    out = np.empty((len(q), 3, 3))
    out[:, 0] = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], 1)
    out[:, 1] = np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], 1)
    out[:, 2] = np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1)
    return out


# -------------------------------------------------------------- projection --
def _geom(params, cam, near):
    """projection.py:77-109 (identity pose delta; the camera is the effective one)."""
    R, t = np.asarray(cam["R"], float), np.asarray(cam["t"], float)
    pc = params["positions"] @ R.T + t
    o = 1.0 / (1.0 + np.exp(-params["opacity_logits"]))
    ids = np.flatnonzero((pc[:, 2] > near) & (o >= MIN_OPACITY))
    X, Y, Z = pc[ids].T
    Rq = _rotmat(params["rotations"][ids]) if len(ids) else np.zeros((0, 3, 3))
    s = np.exp(params["log_scales"][ids])
    M = Rq * s[:, None, :]
    S3 = M @ M.transpose(0, 2, 1)
    J = np.zeros((len(ids), 2, 3))
    J[:, 0, 0] = cam["fx"] / Z
    J[:, 0, 2] = -cam["fx"] * X / Z ** 2
    J[:, 1, 1] = cam["fy"] / Z
    J[:, 1, 2] = -cam["fy"] * Y / Z ** 2
    A = J @ R
    S2 = A @ S3 @ A.transpose(0, 2, 1)
    S2[:, 0, 0] += COV_DILATION
    S2[:, 1, 1] += COV_DILATION
    return dict(R=R, ids=ids, X=X, Y=Y, Z=Z, o=o[ids], Rq=Rq, s=s, M=M, S3=S3, J=J, A=A, S2=S2)


def _sh_basis(deg, d):
    """scene.py:186-221."""
    x, y, z = d.T
    c1 = 0.4886025119029199
    c2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
          -1.0925484305920792, 0.5462742152960396)
    c3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
          -0.4570457994644658, 1.445305721320277, -0.5900435899266435)
    cols = [np.ones_like(x)]
    if deg >= 1:
        cols += [-c1 * y, c1 * z, -c1 * x]
    if deg >= 2:
        xx, yy, zz = x * x, y * y, z * z
        cols += [c2[0] * x * y, c2[1] * y * z, c2[2] * (2 * zz - xx - yy), c2[3] * x * z,
                 c2[4] * (xx - yy)]
    if deg >= 3:
        cols += [c3[0] * y * (3 * xx - yy), c3[1] * x * y * z, c3[2] * y * (4 * zz - xx - yy),
                 c3[3] * z * (2 * zz - 3 * xx - 3 * yy), c3[4] * x * (4 * zz - xx - yy),
                 c3[5] * z * (xx - yy), c3[6] * x * (xx - 3 * yy)]
    return np.stack(cols, 1)


def project(params, cam, near=0.01):
    """project (projection.py:112-136) + per-row colour (trainer.py:170-178).
    Returns (batch, colors)."""
    g = _geom(params, cam, near)
    S2 = g["S2"]
    s11, s12, s22 = S2[:, 0, 0], S2[:, 0, 1], S2[:, 1, 1]
    det = s11 * s22 - s12 * s12
    batch = dict(
        means2d=np.stack([cam["fx"] * g["X"] / g["Z"] + cam["cx"],
                          cam["fy"] * g["Y"] / g["Z"] + cam["cy"]], 1),
        conics=np.stack([s22 / det, -s12 / det, s11 / det], 1),
        level_t=np.maximum(0.0, 2.0 * np.log(255.0 * g["o"])),
        depths=g["Z"].copy(), opacities=g["o"].copy(), source_ids=g["ids"].astype(np.int64),
        width=cam["width"], height=cam["height"])
    coef = params["colors"][g["ids"]]
    C = coef.shape[1]
    if C == 1:
        colors = coef[:, 0, :].copy()
    else:
        center = -g["R"].T @ np.asarray(cam["t"], float)
        v = params["positions"][g["ids"]] - center
        d = v / np.linalg.norm(v, axis=1, keepdims=True)
        colors = np.einsum("nc,ncd->nd", _sh_basis(int(round(np.sqrt(C))) - 1, d), coef)
    return batch, colors


# ---------------------------------------------------------------- binning --
def _span(lo, hi, n_tiles):
    """binning.py:74-84."""
    t0 = np.maximum(np.ceil(np.asarray(lo) / TILE - 1.0).astype(np.int64), 0)
    t1 = np.minimum(np.floor(np.asarray(hi) / TILE).astype(np.int64), n_tiles - 1)
    return t0, t1


def _tiles(batch):
    return -(-batch["width"] // TILE), -(-batch["height"] // TILE)


def snugboxes(batch):
    """compute_snugboxes (binning.py:87-104) -> (x_min, x_max, y_min, y_max, rect)."""
    a, b, c = batch["conics"].T
    t = batch["level_t"]
    det = a * c - b * b
    ex = np.sqrt(c * t / det)
    ey = np.sqrt(a * t / det)
    mx, my = batch["means2d"].T
    tiles_x, tiles_y = _tiles(batch)
    x0, x1 = _span(mx - ex, mx + ex, tiles_x)
    y0, y1 = _span(my - ey, my + ey, tiles_y)
    return mx - ex, mx + ex, my - ey, my + ey, np.stack([x0, x1, y0, y1], 1)


def _finish_index(splat_rows, tile_ids, batch):
    """Keys, stable order (key, then emission row) and ranges (binning.py:137-158)."""
    tiles_x, tiles_y = _tiles(batch)
    depth_bits = np.asarray(batch["depths"], np.float32).view(np.uint32).astype(np.uint64)
    keys = (tile_ids.astype(np.uint64) << np.uint64(32)) | depth_bits[splat_rows]
    order = np.lexsort((splat_rows, keys))
    keys = keys[order]
    values = splat_rows[order].astype(np.int64)
    offsets = np.searchsorted((keys >> np.uint64(32)).astype(np.int64),
                              np.arange(tiles_x * tiles_y + 1))
    return dict(keys=keys, values=values, offsets=offsets.astype(np.int64),
                tiles_x=tiles_x, tiles_y=tiles_y)


def bin_sequential(batch):
    """Column walk (binning.py:166-222), iterated column-offset-major."""
    tiles_x, tiles_y = _tiles(batch)
    x_min, x_max, _, _, rect = snugboxes(batch)
    a, b, c = batch["conics"].T
    t = batch["level_t"]
    mx, my = batch["means2d"].T
    ncols = np.maximum(0, rect[:, 1] - rect[:, 0] + 1)
    rows_out, tiles_out = [], []
    for j in range(int(ncols.max()) if len(ncols) else 0):
        s = np.flatnonzero(ncols > j)
        tx = rect[s, 0] + j
        A, B, Cc, Tt, MX = a[s], b[s], c[s], t[s], mx[s]
        det = A * Cc - B * B
        xl = np.maximum(TILE * tx, x_min[s]) - MX
        xr = np.minimum(TILE * tx + TILE, x_max[s]) - MX

        def ybounds(dx):
            rad = np.sqrt(np.maximum(0.0, (B * B - A * Cc) * dx * dx + Tt * Cc))
            return (-B * dx - rad) / Cc, (-B * dx + rad) / Cc

        lo_l, hi_l = ybounds(xl)
        lo_r, hi_r = ybounds(xr)
        ylo, yhi = np.minimum(lo_l, lo_r), np.maximum(hi_l, hi_r)
        ymax_rel = np.sqrt(A * Tt / det)
        dx_up = -(B / A) * ymax_rel
        dx_dn = -dx_up
        yhi = np.where((dx_up >= xl) & (dx_up <= xr), np.maximum(yhi, ymax_rel), yhi)
        ylo = np.where((dx_dn >= xl) & (dx_dn <= xr), np.minimum(ylo, -ymax_rel), ylo)
        r0, r1 = _span(ylo + my[s], yhi + my[s], tiles_y)
        r0 = np.maximum(r0, rect[s, 2])
        r1 = np.minimum(r1, rect[s, 3])
        for k in range(int(np.max(r1 - r0 + 1, initial=0))):
            hit = r1 - r0 >= k
            rows_out.append(s[hit])
            tiles_out.append((r0[hit] + k) * tiles_x + tx[hit])
    if not rows_out:
        return _finish_index(np.empty(0, np.int64), np.empty(0, np.int64), batch)
    return _finish_index(np.concatenate(rows_out), np.concatenate(tiles_out), batch)


def min_q_box(conics, rx0, rx1, ry0, ry1):
    """Exact min of the quadratic over a closed box (binning.py:241-259)."""
    a, b, c = conics.T
    inside = (rx0 <= 0.0) & (0.0 <= rx1) & (ry0 <= 0.0) & (0.0 <= ry1)

    def q(dx, dy):
        return a * dx * dx + 2.0 * b * dx * dy + c * dy * dy

    yx0 = np.clip(-(b / c) * rx0, ry0, ry1)
    yx1 = np.clip(-(b / c) * rx1, ry0, ry1)
    xy0 = np.clip(-(b / a) * ry0, rx0, rx1)
    xy1 = np.clip(-(b / a) * ry1, rx0, rx1)
    m = np.minimum(np.minimum(q(rx0, yx0), q(rx1, yx1)), np.minimum(q(xy0, ry0), q(xy1, ry1)))
    return np.where(inside, 0.0, m)


def bin_load_balanced(batch):
    """Candidate-rect min-q test (binning.py:262-286)."""
    _, _, _, _, rect = snugboxes(batch)
    tiles_x, _ = _tiles(batch)
    ncols = np.maximum(0, rect[:, 1] - rect[:, 0] + 1)
    nrows = np.maximum(0, rect[:, 3] - rect[:, 2] + 1)
    cnt = ncols * nrows
    splat = np.repeat(np.arange(len(cnt)), cnt)
    within = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    tx = rect[splat, 0] + within // np.maximum(nrows[splat], 1)
    ty = rect[splat, 2] + within % np.maximum(nrows[splat], 1)
    mx, my = batch["means2d"][splat].T
    rx0 = TILE * tx - mx
    ry0 = TILE * ty - my
    hit = min_q_box(batch["conics"][splat], rx0, rx0 + TILE, ry0, ry0 + TILE) \
        <= batch["level_t"][splat]
    return _finish_index(splat[hit], ty[hit] * tiles_x + tx[hit], batch)


def checksum(index):
    """TileIndex.checksum (binning.py:67-71)."""
    h = hashlib.sha256()
    h.update(np.asarray(index["keys"], np.uint64).tobytes())
    h.update(np.asarray(index["values"], np.int64).tobytes())
    return h.hexdigest()[:16]


# ----------------------------------------------------------------- render --
def _tile_pixels(tile, tiles_x, width, height):
    ty, tx = divmod(tile, tiles_x)
    x0, y0 = tx * TILE, ty * TILE
    x1, y1 = min(x0 + TILE, width), min(y0 + TILE, height)
    gy, gx = np.mgrid[y0:y1, x0:x1]
    return (x0, y0, x1, y1), gx.reshape(-1) + 0.5, gy.reshape(-1) + 0.5


def _alpha(batch, row, px, py):
    """splat_alpha (forward.py:71-84)."""
    a, b, c = batch["conics"][row]
    dx = px - batch["means2d"][row, 0]
    dy = py - batch["means2d"][row, 1]
    q = a * dx * dx + 2.0 * b * (dx * dy) + c * dy * dy
    gauss = np.exp(-0.5 * q)
    raw = batch["opacities"][row] * gauss
    return np.minimum(ALPHA_CAP, raw), raw, gauss, dx, dy


def render(batch, index, colors, background, record_checkpoints=True, tiles=None):
    """Front-to-back compositing with 32-position checkpoints (forward.py:87-161).
    checkpoints[tile] is (G, 5, npix) over the tile's pixels row-major.
    `tiles` optionally restricts the tiles processed (bounded CPU samples)."""
    W, H = batch["width"], batch["height"]
    bg = np.asarray(background, float).reshape(3)
    out = dict(color=np.empty((H, W, 3)), depth=np.zeros((H, W)), final_T=np.ones((H, W)),
               n_contrib=np.zeros((H, W), np.int32), n_considered=np.zeros((H, W), np.int32),
               checkpoints={})
    out["color"][:] = bg
    offs, vals = index["offsets"], index["values"]
    todo = range(index["tiles_x"] * index["tiles_y"]) if tiles is None else tiles
    for tile in todo:
        lo, hi = int(offs[tile]), int(offs[tile + 1])
        if lo == hi:
            continue
        (x0, y0, x1, y1), px, py = _tile_pixels(tile, index["tiles_x"], W, H)
        npx = px.size
        T = np.ones(npx)
        C = np.zeros((npx, 3))
        D = np.zeros(npx)
        nb = np.zeros(npx, np.int32)
        nc = np.zeros(npx, np.int32)
        alive = np.ones(npx, bool)
        want = (hi - lo) // GROUP
        recs = []
        for k in range(hi - lo):
            row = vals[lo + k]
            al = _alpha(batch, row, px, py)[0]
            bl = alive & (al >= MIN_OPACITY)
            w = np.where(bl, T * al, 0.0)
            C += w[:, None] * colors[row]
            D += w * batch["depths"][row]
            T = np.where(bl, T * (1.0 - al), T)
            nb += bl
            nc[alive] = k + 1
            alive &= T >= T_TERMINATE
            if record_checkpoints and (k + 1) % GROUP == 0:
                recs.append(np.concatenate([T[None], C.T, D[None]]))
            if not alive.any():
                while record_checkpoints and len(recs) < want:
                    recs.append(np.concatenate([T[None], C.T, D[None]]))
                break
        shp = (y1 - y0, x1 - x0)
        out["color"][y0:y1, x0:x1] = (C + T[:, None] * bg).reshape(shp + (3,))
        out["depth"][y0:y1, x0:x1] = D.reshape(shp)
        out["final_T"][y0:y1, x0:x1] = T.reshape(shp)
        out["n_contrib"][y0:y1, x0:x1] = nb.reshape(shp)
        out["n_considered"][y0:y1, x0:x1] = nc.reshape(shp)
        if recs:
            out["checkpoints"][tile] = np.stack(recs)
    return out


# --------------------------------------------------------------- backward --
def backward_per_gaussian(bufs, batch, index, colors, grad_color, grad_depth=None,
                          grad_final_T=None, tiles=None):
    """Group replay from checkpoints (backward.py:137-223).  `tiles` optionally
    restricts the tiles processed (bounded CPU-baseline samples).
    Returns dict d_means2d, d_conics, d_opacities, d_colors, d_depths, merges."""
    M = len(batch["depths"])
    out = dict(d_means2d=np.zeros((M, 2)), d_conics=np.zeros((M, 3)), d_opacities=np.zeros(M),
               d_colors=np.zeros((M, 3)), d_depths=np.zeros(M), merges=0)
    W, H = batch["width"], batch["height"]
    offs, vals = index["offsets"], index["values"]
    todo = range(index["tiles_x"] * index["tiles_y"]) if tiles is None else tiles
    for tile in todo:
        lo, hi = int(offs[tile]), int(offs[tile + 1])
        if lo == hi:
            continue
        (x0, y0, x1, y1), px, py = _tile_pixels(tile, index["tiles_x"], W, H)
        gc = grad_color[y0:y1, x0:x1].reshape(-1, 3)
        gd = None if grad_depth is None else grad_depth[y0:y1, x0:x1].reshape(-1)
        gt = None if grad_final_T is None else grad_final_T[y0:y1, x0:x1].reshape(-1)
        if not (np.any(gc) or (gd is not None and np.any(gd)) or (gt is not None and np.any(gt))):
            continue
        n = hi - lo
        ck = bufs["checkpoints"].get(tile)
        if n > GROUP and (ck is None or len(ck) < n // GROUP):
            raise RuntimeError(f"tile {tile}: checkpoints missing")
        ncons = bufs["n_considered"][y0:y1, x0:x1].reshape(-1)
        fT = bufs["final_T"][y0:y1, x0:x1].reshape(-1)
        ctot = bufs["color"][y0:y1, x0:x1].reshape(-1, 3)
        dtot = bufs["depth"][y0:y1, x0:x1].reshape(-1)
        tf_term = None if gt is None else -gt * fT
        # groups past the tile's largest n_considered contribute nothing
        # (part is all False there: backward.py:189 skips them one position
        # at a time); bounding the walk keeps heavy C3 tiles (200k entries)
        # affordable.  merges still counts every pair (backward.py:214-222).
        n_walk = min(n, int(ncons.max(initial=0)))
        for g in range(-(-n_walk // GROUP)):
            p0, p1 = g * GROUP, min(n, (g + 1) * GROUP)
            if g == 0:
                T, C, D = np.ones(px.size), np.zeros((px.size, 3)), np.zeros(px.size)
            else:
                st = ck[g - 1]
                T, C, D = st[0].copy(), st[1:4].T.copy(), st[4].copy()
            for p in range(p0, p1):
                row = vals[lo + p]
                al, raw, gauss, dx, dy = _alpha(batch, row, px, py)
                part = (p < ncons) & (al >= MIN_OPACITY)
                if not part.any():
                    continue
                om = 1.0 - al
                w = np.where(part, T * al, 0.0)
                Ca = C + w[:, None] * colors[row]
                Da = D + w * batch["depths"][row]
                dLda = np.sum(gc * (T[:, None] * colors[row] - (ctot - Ca) / om[:, None]), 1)
                if gd is not None:
                    dLda += gd * (T * batch["depths"][row] - (dtot - Da) / om)
                if tf_term is not None:
                    dLda += tf_term / om
                dLda = np.where(part, dLda, 0.0)
                capped = raw > al
                gq = np.where(capped, 0.0, -0.5 * dLda * al)
                a, b, c = batch["conics"][row]
                out["d_conics"][row] += [np.sum(gq * dx * dx), np.sum(gq * 2.0 * dx * dy),
                                         np.sum(gq * dy * dy)]
                out["d_means2d"][row] += [np.sum(gq * (-2.0 * a * dx - 2.0 * b * dy)),
                                          np.sum(gq * (-2.0 * b * dx - 2.0 * c * dy))]
                out["d_opacities"][row] += np.sum(np.where(capped, 0.0, dLda * gauss))
                out["d_colors"][row] += w @ gc
                if gd is not None:
                    out["d_depths"][row] += np.sum(gd * w)
                T = np.where(part, T * om, T)
                C, D = Ca, Da
        out["merges"] += n  # one merge per (splat, tile) pair of a processed tile
    return out


# ------------------------------------------------------------- projection vjp
def project_vjp(params, cam, batch, g2, near=0.01):
    """Chain 2D gradients to 3D parameters (projection.py:139-241; identity pose
    delta) plus the SH-0 colour copy (trainer.py:240-241).  Returns dict of
    positions, log_scales, rotations, opacity_logits, colors and pose sums."""
    g = _geom(params, cam, near)
    ids = g["ids"]
    N = len(params["positions"])
    out = dict(positions=np.zeros((N, 3)), log_scales=np.zeros((N, 3)),
               rotations=np.zeros((N, 4)), opacity_logits=np.zeros(N),
               colors=np.zeros_like(params["colors"]))
    if len(ids) == 0:
        return out
    fx, fy = cam["fx"], cam["fy"]
    X, Y, Z, A, J, S3, M, Rq, s, R = (g[k] for k in ("X", "Y", "Z", "A", "J", "S3", "M", "Rq",
                                                     "s", "R"))
    con = batch["conics"]
    Cm = np.stack([np.stack([con[:, 0], con[:, 1]], 1), np.stack([con[:, 1], con[:, 2]], 1)], 1)
    gcon = g2["d_conics"]
    Gb = np.stack([np.stack([gcon[:, 0], 0.5 * gcon[:, 1]], 1),
                   np.stack([0.5 * gcon[:, 1], gcon[:, 2]], 1)], 1)
    GS = -Cm @ Gb @ Cm
    GA = 2.0 * (GS @ A @ S3)
    GS3 = A.transpose(0, 2, 1) @ GS @ A
    GJ = GA @ R.T
    iz = 1.0 / Z
    iz2 = iz * iz
    gm = g2["d_means2d"]
    gp = np.zeros((len(ids), 3))
    gp[:, 0] = gm[:, 0] * fx * iz - GJ[:, 0, 2] * fx * iz2
    gp[:, 1] = gm[:, 1] * fy * iz - GJ[:, 1, 2] * fy * iz2
    gp[:, 2] = (-gm[:, 0] * fx * X * iz2 - gm[:, 1] * fy * Y * iz2 + g2["d_depths"]
                - GJ[:, 0, 0] * fx * iz2 - GJ[:, 1, 1] * fy * iz2
                + GJ[:, 0, 2] * 2.0 * fx * X * iz2 * iz + GJ[:, 1, 2] * 2.0 * fy * Y * iz2 * iz)
    GM = 2.0 * (GS3 @ M)
    GR = GM * s[:, None, :]
    out["log_scales"][ids] = np.einsum("mij,mij->mj", GM, Rq) * s
    qraw = params["rotations"][ids]
    qn = np.linalg.norm(qraw, axis=1, keepdims=True)
    w, x, y, z = (qraw / qn).T
    zero = np.zeros_like(w)
    basis = [np.stack([zero, -z, y, z, zero, -x, -y, x, zero], 1),
             np.stack([zero, y, z, y, -2 * x, -w, z, w, -2 * x], 1),
             np.stack([-2 * y, x, w, x, zero, z, -w, z, -2 * y], 1),
             np.stack([-2 * z, -w, x, w, -2 * z, y, x, y, zero], 1)]
    gq = np.stack([2.0 * np.sum(GR.reshape(-1, 9) * bk, 1) for bk in basis], 1)
    qh = qraw / qn
    out["rotations"][ids] = (gq - np.sum(gq * qh, 1, keepdims=True) * qh) / qn
    out["positions"][ids] = gp @ R
    o = batch["opacities"]
    out["opacity_logits"][ids] = g2["d_opacities"] * o * (1.0 - o)
    out["colors"][ids, 0, :] = g2["d_colors"]
    out["pose_S1"] = (J.transpose(0, 2, 1) @ GA).sum(0) + gp.T @ params["positions"][ids]
    out["pose_S2"] = gp.sum(0)
    return out


# ------------------------------------------------------------------- Adam --
def adam_step(p, g, m, v, t, lr, renormalize=False):
    """One bias-corrected dense Adam step on row-major arrays (optim.py:60-88);
    rows with a non-finite gradient are skipped.  Returns skipped row count."""
    b1, b2, eps = 0.9, 0.999, 1e-15
    rows = len(p)
    ok = np.isfinite(g.reshape(rows, -1)).all(1)
    m[ok] = b1 * m[ok] + (1 - b1) * g[ok]
    v[ok] = b2 * v[ok] + (1 - b2) * g[ok] ** 2
    p[ok] -= lr * (m[ok] / (1 - b1 ** t)) / (np.sqrt(v[ok] / (1 - b2 ** t)) + eps)
    if renormalize:
        nrm = np.linalg.norm(p[ok], axis=1, keepdims=True)
        p[ok] = np.divide(p[ok], nrm, where=nrm > 0)
    return int((~ok).sum())


# ------------------------------------------------------------------- loss --
_WIN = np.exp(-((np.arange(11) - 5.0) ** 2) / (2.0 * 1.5 ** 2))
_WIN /= _WIN.sum()


def _blur(img):
    return correlate1d(correlate1d(img, _WIN, axis=0, mode="constant"), _WIN, axis=1,
                       mode="constant")


def photometric(rendered, gt, lam=0.2):
    """(1 - lam) L1 + lam (1 - SSIM) and its gradient (losses.py:44-91)."""
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    diff = rendered - gt
    l1 = float(np.abs(diff).mean())
    m1, m2 = _blur(rendered), _blur(gt)
    s1 = _blur(rendered * rendered) - m1 * m1
    s2 = _blur(gt * gt) - m2 * m2
    s12 = _blur(rendered * gt) - m1 * m2
    A1, A2 = 2 * m1 * m2 + c1, 2 * s12 + c2
    B1, B2 = m1 * m1 + m2 * m2 + c1, s1 + s2 + c2
    smap = A1 * A2 / (B1 * B2)
    ssim = float(smap.mean())
    k = 1.0 / smap.size
    dA1, dA2 = k * A2 / (B1 * B2), k * A1 / (B1 * B2)
    dB1, dB2 = -k * A1 * A2 / (B1 * B1 * B2), -k * A1 * A2 / (B1 * B2 * B2)
    gmu = 2 * m2 * (dA1 - dA2) + 2 * m1 * (dB1 - dB2)
    gssim = _blur(gmu) + _blur(dB2) * 2.0 * rendered + _blur(2.0 * dA2) * gt
    e = (1 - lam) * l1 + lam * (1 - ssim)
    grad = (1 - lam) * np.sign(diff) / diff.size - lam * gssim
    return e, l1, ssim, grad


def pose_from_sums(S1, S2, R_cam):
    """Pose gradient at an identity delta from the reduced sums
    (projection.py:232-240: J_l(0) = I)."""
    R_cam = np.asarray(R_cam, float)
    B = (R_cam.T @ S1).T
    rot = np.array([B[1, 2] - B[2, 1], B[2, 0] - B[0, 2], B[0, 1] - B[1, 0]])
    return rot, R_cam.T @ S2
