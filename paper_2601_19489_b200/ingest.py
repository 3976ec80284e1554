"""Scene container and PLY splat checkpoints (reference: tilesplat/ingest.py;
SURVEY.md §8(f) #4).

`write_ply` / `read_ply` keep the reference's on-disk format exactly
(ingest.py:262-344): binary little-endian PLY, one `double` property per
column in the order x y z f_dc_0..2 f_rest_* opacity scale_0..2 rot_0..3,
f_rest flattened channel-major.  A file written by the reference loads here
(values rounded to the device's FP32) and a file written here loads in the
reference; read(write(s)) is bit-for-bit for any FP32 set.  The device set
is copied to the host once per file (one D2H of 14+ floats per splat).
COLMAP parsing, image decoding and depth alignment are the reference's
offline data path and are not rebuilt.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .scene import Camera, GaussianSet


class PlySchemaError(ValueError):
    """Malformed or unsupported splat PLY (ingest.py:36-37)."""


@dataclass
class Scene:
    """Everything the trainer needs (ingest.py:54-62): posed cameras with
    ground truth, seed points, and the scene extent."""
    cameras: list
    points: np.ndarray
    colors: np.ndarray
    extent: float
    warnings: list = field(default_factory=list)


# On-disk column order of a splat PLY (the reference's format, ingest.py:270-
# 288): position, DC colour, the higher SH coefficients flattened channel-
# major, opacity logit, log scales, quaternion (w, x, y, z).  Each entry is
# (property name, GaussianSet field, column index inside that field).
def _ply_columns(n_coeffs: int) -> list[tuple[str, str, tuple]]:
    cols = [(axis, "positions", (i,)) for i, axis in enumerate("xyz")]
    cols += [(f"f_dc_{ch}", "colors", (0, ch)) for ch in range(3)]
    higher = n_coeffs - 1
    cols += [(f"f_rest_{ch * higher + k}", "colors", (k + 1, ch))
             for ch in range(3) for k in range(higher)]
    cols.append(("opacity", "opacity_logits", ()))
    cols += [(f"scale_{i}", "log_scales", (i,)) for i in range(3)]
    cols += [(f"rot_{i}", "rotations", (i,)) for i in range(4)]
    return cols


def write_ply(gset: GaussianSet, path) -> None:
    """Binary little-endian PLY, one double per property (ingest.py:270-288)."""
    host = gset.to_numpy()
    n = len(gset)
    cols = _ply_columns(host["colors"].shape[1])
    table = np.empty((n, len(cols)), dtype="<f8")
    for j, (_, field_name, idx) in enumerate(cols):
        src = host[field_name]
        table[:, j] = src if not idx else src[(slice(None),) + idx]
    head = "".join(f"property double {name}\n" for name, _, _ in cols)
    preamble = (f"ply\nformat binary_little_endian 1.0\nelement vertex {n}\n{head}"
                "end_header\n").encode()
    with open(path, "wb") as fh:
        fh.write(preamble)
        fh.write(table.tobytes())


_PLY_SCALARS = {"float": "<f4", "float32": "<f4", "double": "<f8", "float64": "<f8"}


def _parse_ply_header(fh, path):
    """(vertex count, [(property, numpy dtype)]) of a binary little-endian
    vertex-only PLY; the file position is left at the first vertex byte."""
    if fh.readline().rstrip(b"\r\n") != b"ply":
        raise PlySchemaError(f"{path}: missing 'ply' magic")
    count, fields = None, []
    for raw in iter(fh.readline, b""):
        words = raw.decode("ascii", "replace").split()
        if not words:
            continue
        key = words[0]
        if key == "end_header":
            if count is None:
                raise PlySchemaError(f"{path}: no vertex element declared")
            return count, fields
        if key == "format" and words[1:2] != ["binary_little_endian"]:
            raise PlySchemaError(f"{path}: only binary_little_endian PLY is supported, "
                                 f"got {' '.join(words[1:])}")
        elif key == "element":
            if words[1] != "vertex":
                raise PlySchemaError(f"{path}: element '{words[1]}' is not supported")
            count = int(words[2])
        elif key == "property":
            if words[1] not in _PLY_SCALARS:
                raise PlySchemaError(f"{path}: property type '{words[1]}' is not supported")
            fields.append((words[2], _PLY_SCALARS[words[1]]))
    raise PlySchemaError(f"{path}: header never ends")


def read_ply(path) -> GaussianSet:
    """Load a splat PLY written by the reference or by write_ply; float and
    double properties are both accepted (ingest.py:291-344)."""
    with open(path, "rb") as fh:
        count, fields = _parse_ply_header(fh, path)
        rec = np.dtype(fields)
        body = np.frombuffer(fh.read(rec.itemsize * count), dtype=rec, count=count)
    present = set(rec.names or ())
    higher_terms = sum(1 for name in present if name.startswith("f_rest_"))
    if higher_terms % 3 != 0:
        raise PlySchemaError(f"{path}: {higher_terms} f_rest properties is not a multiple of 3")
    n_coeffs = 1 + higher_terms // 3
    cols = _ply_columns(n_coeffs)
    absent = [name for name, _, _ in cols if name not in present]
    if absent:
        raise PlySchemaError(f"{path}: required properties absent: {', '.join(absent)}")
    shapes = {"positions": (count, 3), "log_scales": (count, 3), "rotations": (count, 4),
              "opacity_logits": (count,), "colors": (count, n_coeffs, 3)}
    out = {k: np.empty(v, dtype=np.float64) for k, v in shapes.items()}
    for name, field_name, idx in cols:
        out[field_name][(slice(None),) + idx] = body[name]
    return GaussianSet(**out)


__all__ = ["Camera", "PlySchemaError", "Scene", "read_ply", "write_ply"]
