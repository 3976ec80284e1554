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


def _ply_property_names(n_coeffs: int) -> list[str]:
    names = ["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2"]
    names += [f"f_rest_{i}" for i in range(3 * (n_coeffs - 1))]
    names += ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]
    return names


def write_ply(gset: GaussianSet, path) -> None:
    """Binary little-endian PLY, double precision (ingest.py:270-288)."""
    n = len(gset)
    h = gset.to_numpy()
    colors = h["colors"]
    n_coeffs = colors.shape[1]
    names = _ply_property_names(n_coeffs)
    rest = np.transpose(colors[:, 1:, :], (0, 2, 1)).reshape(n, 3 * (n_coeffs - 1))
    data = np.empty((n, len(names)), dtype="<f8")
    data[:, 0:3] = h["positions"]
    data[:, 3:6] = colors[:, 0, :]
    c = 6 + rest.shape[1]
    data[:, 6:c] = rest
    data[:, c] = h["opacity_logits"]
    data[:, c + 1:c + 4] = h["log_scales"]
    data[:, c + 4:c + 8] = h["rotations"]
    header = ["ply", "format binary_little_endian 1.0", f"element vertex {n}"]
    header += [f"property double {name}" for name in names]
    header.append("end_header")
    with open(path, "wb") as fh:
        fh.write(("\n".join(header) + "\n").encode())
        fh.write(np.ascontiguousarray(data).tobytes())


def read_ply(path) -> GaussianSet:
    """Read a splat PLY; float or double properties (ingest.py:291-344)."""
    with open(path, "rb") as fh:
        if fh.readline().strip() != b"ply":
            raise PlySchemaError(f"{path}: not a PLY file")
        n = None
        props: list[tuple[str, str]] = []
        while True:
            line = fh.readline()
            if not line:
                raise PlySchemaError(f"{path}: unterminated header")
            tokens = line.decode().strip().split()
            if not tokens:
                continue
            if tokens[0] == "format" and tokens[1] != "binary_little_endian":
                raise PlySchemaError(f"{path}: unsupported format {tokens[1]}")
            if tokens[0] == "element":
                if tokens[1] != "vertex":
                    raise PlySchemaError(f"{path}: unexpected element {tokens[1]}")
                n = int(tokens[2])
            if tokens[0] == "property":
                props.append((tokens[2], tokens[1]))
            if tokens[0] == "end_header":
                break
        if n is None:
            raise PlySchemaError(f"{path}: missing vertex element")
        typemap = {"float": "<f4", "float32": "<f4", "double": "<f8", "float64": "<f8"}
        try:
            dtype = np.dtype([(name, typemap[t]) for name, t in props])
        except KeyError as exc:
            raise PlySchemaError(f"{path}: unsupported property type {exc}") from exc
        raw = np.frombuffer(fh.read(dtype.itemsize * n), dtype=dtype, count=n)
    have = {name for name, _ in props}
    n_rest = len([name for name in have if name.startswith("f_rest_")])
    if n_rest % 3:
        raise PlySchemaError(f"{path}: f_rest count {n_rest} not divisible by 3")
    n_coeffs = n_rest // 3 + 1
    for required in _ply_property_names(n_coeffs):
        if required not in have:
            raise PlySchemaError(f"{path}: missing property \"{required}\"")

    def col(name):
        return raw[name].astype(np.float64)

    positions = np.stack([col("x"), col("y"), col("z")], axis=1)
    colors = np.empty((n, n_coeffs, 3))
    colors[:, 0, :] = np.stack([col(f"f_dc_{i}") for i in range(3)], axis=1)
    for ch in range(3):
        for j in range(n_coeffs - 1):
            colors[:, j + 1, ch] = col(f"f_rest_{ch * (n_coeffs - 1) + j}")
    log_scales = np.stack([col(f"scale_{i}") for i in range(3)], axis=1)
    rotations = np.stack([col(f"rot_{i}") for i in range(4)], axis=1)
    return GaussianSet(positions, log_scales, rotations, col("opacity"), colors)


__all__ = ["Camera", "PlySchemaError", "Scene", "read_ply", "write_ply"]
