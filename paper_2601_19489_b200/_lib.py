"""ctypes binding of the sm_100a C-ABI library (include/tilesplat_b200.h).

The product path has exactly one implementation: the CUDA kernels in
libtilesplat_b200.so.  There is no CPU fallback; if the library is missing or
no CUDA device is visible, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

_HERE = Path(__file__).resolve().parent
# TSR_LIB overrides the path (instrumented builds for profiling only)
LIB_PATH = Path(os.environ.get("TSR_LIB", _HERE / "libtilesplat_b200.so"))

TSR_OK = 0
TSR_E_INVALID = 1
TSR_E_CUDA = 2
TSR_E_CAPACITY = 3
TSR_E_WORKSPACE = 4
REC_FLOATS = 12
GRAD2D_FLOATS = 10
MAX_ADAM_GROUPS = 8

c_i32, c_i64, c_f32, c_vp, c_sz = (ctypes.c_int32, ctypes.c_int64, ctypes.c_float,
                                   ctypes.c_void_p, ctypes.c_size_t)


class Camera_t(ctypes.Structure):
    _fields_ = [("fx", c_f32), ("fy", c_f32), ("cx", c_f32), ("cy", c_f32),
                ("width", c_i32), ("height", c_i32), ("R", c_f32 * 9), ("t", c_f32 * 3),
                ("center", c_f32 * 3), ("near_plane", c_f32)]


class Gaussians_t(ctypes.Structure):
    _fields_ = [("positions", c_vp), ("log_scales", c_vp), ("rotations", c_vp),
                ("opacity_logits", c_vp), ("colors", c_vp), ("n", c_i64),
                ("sh_coeffs", c_i32)]


class AdamGroup_t(ctypes.Structure):
    _fields_ = [("param", c_vp), ("grad", c_vp), ("exp_avg", c_vp), ("exp_avg_sq", c_vp),
                ("rows", c_i64), ("width", c_i32), ("renormalize", c_i32), ("lr", c_f32),
                ("bias_correction1", c_f32), ("bias_correction2", c_f32)]


# name -> (restype, argtypes); mirrors include/tilesplat_b200.h
_SIGNATURES = {
    "tsr_preprocess_workspace": (c_sz, [c_i64]),
    "tsr_preprocess_fwd": (c_i32, [ctypes.POINTER(Gaussians_t), ctypes.POINTER(Camera_t), c_i32,
                                   c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "tsr_count_pairs": (c_i32, [c_vp, c_i64, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsr_snugboxes": (c_i32, [c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsr_index_workspace": (c_sz, [c_i64, c_i64]),
    "tsr_build_index": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_i32, c_i32,
                                c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "tsr_render_score": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, ctypes.POINTER(c_f32), c_i32,
                                 c_vp, c_f32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                 c_vp, c_vp, c_vp]),
    "tsr_render_fwd": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, ctypes.POINTER(c_f32), c_vp, c_vp,
                               c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsr_render_fwd_ex": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, ctypes.POINTER(c_f32), c_vp,
                                  c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "tsr_render_bwd": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp,
                               c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsr_render_bwd_det": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp,
                                   c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                   c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "tsr_tile_order": (c_i32, [c_vp, c_i32, c_vp, c_vp]),
    "tsr_render_fwd_ordered": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, ctypes.POINTER(c_f32),
                                       c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp,
                                       c_vp]),
    "tsr_render_bwd_ordered": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp,
                                       c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsr_render_bwd_adam": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp,
                                    c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                    ctypes.POINTER(Gaussians_t), ctypes.POINTER(Camera_t),
                                    ctypes.POINTER(AdamGroup_t), c_vp, c_vp, c_vp, c_vp, c_vp,
                                    c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsr_render_bwd_workspace": (c_sz, [c_i32, c_i32, c_i64]),
    "tsr_render_fwd_regions": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, ctypes.POINTER(c_f32),
                                       c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                       c_vp, c_vp, c_i32, c_vp, c_vp]),
    "tsr_region_list_entries": (c_sz, [c_i32, c_i32, c_i64]),
    "tsr_region_seg_entries": (c_sz, [c_i32, c_i32, c_i64]),
    "tsr_region_unit_entries": (c_sz, [c_i32, c_i32, c_i64]),
    "tsr_region_ctl_entries": (c_sz, []),
    "tsr_render_bwd_regions": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp,
                                       c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                       c_vp, c_vp, c_i32, c_vp]),
    "tsr_render_bwd_ws": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp,
                                  c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_sz, c_vp]),
    "tsr_render_bwd_ws_det": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp,
                                      c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                      c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_sz,
                                      c_vp]),
    "tsr_build_index_det": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_i32,
                                    c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp, c_vp,
                                    c_vp, c_vp, c_vp]),
    "tsr_preprocess_bwd": (c_i32, [ctypes.POINTER(Gaussians_t), ctypes.POINTER(Camera_t), c_vp,
                                   c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "tsr_adam_step": (c_i32, [ctypes.POINTER(AdamGroup_t), c_i32, c_vp, c_vp]),
    "tsr_adam_step_dev": (c_i32, [ctypes.POINTER(AdamGroup_t), c_i32, c_vp, c_i32, c_vp, c_vp]),
    "tsr_zero1_peer_adam": (c_i32, [ctypes.POINTER(AdamGroup_t), c_i32, c_i32, c_vp, c_vp,
                                    c_i64, c_i64, c_vp, c_vp]),
    "tsr_preprocess_bwd_adam": (c_i32, [ctypes.POINTER(Gaussians_t), ctypes.POINTER(Camera_t),
                                        c_vp, c_vp, c_vp, ctypes.POINTER(AdamGroup_t), c_vp,
                                        c_vp, c_vp]),
    "tsr_preprocess_bwd_adam_dev": (c_i32, [ctypes.POINTER(Gaussians_t),
                                            ctypes.POINTER(Camera_t), c_vp, c_vp, c_vp,
                                            ctypes.POINTER(AdamGroup_t), c_vp, c_vp, c_vp, c_vp]),
    "tsr_preprocess_bwd_adam_ex": (c_i32, [ctypes.POINTER(Gaussians_t),
                                           ctypes.POINTER(Camera_t), c_vp, c_vp, c_vp,
                                           ctypes.POINTER(AdamGroup_t), c_vp, c_vp, c_vp, c_vp,
                                           c_vp, c_vp, c_vp]),
    "tsr_depth_chain_workspace": (c_sz, []),
    "tsr_depth_chain": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_f32, c_vp, c_vp,
                                c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "tsr_photometric_workspace": (c_sz, [c_i32, c_i32]),
    "tsr_photometric": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_f32, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "tsr_version": (ctypes.c_char_p, []),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None


class NativeLibraryError(RuntimeError):
    """The CUDA library is missing, failed to load, or a call failed."""


def load(require_cuda: bool = True):
    """Load (once) and return the ctypes library handle."""
    global _lib
    if require_cuda and not torch.cuda.is_available():
        raise NativeLibraryError(
            "tilesplat_b200 needs a CUDA device (sm_100a); no CPU fallback exists")
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeLibraryError(
                f"{LIB_PATH} not built; run `make` (or __graft_entry__.build())")
        lib = ctypes.CDLL(os.fspath(LIB_PATH))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(code: int, what: str) -> None:
    if code != TSR_OK:
        names = {1: "invalid argument", 2: "CUDA error", 3: "capacity", 4: "workspace"}
        detail = ""
        if code == TSR_E_CUDA:
            detail = f" ({torch.cuda.current_stream()})"
        raise NativeLibraryError(f"{what} failed: {names.get(code, code)}{detail}")


def ptr(t) -> int | None:
    """Raw device pointer of a tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
