"""The C-ABI library loads without a GPU and exports every symbol that
include/tilesplat_b200.h declares (no compute calls)."""

import ctypes
import re

import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "tilesplat_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|size_t|const char\*)\s+(tsr_\w+)\(", text, re.M)))


def test_header_declares_the_pipeline():
    names = declared_symbols()
    for required in ("tsr_preprocess_fwd", "tsr_count_pairs", "tsr_build_index",
                     "tsr_render_fwd", "tsr_render_bwd", "tsr_photometric",
                     "tsr_preprocess_bwd", "tsr_adam_step", "tsr_preprocess_bwd_adam"):
        assert required in names


def test_library_exports_every_declared_symbol():
    import torch  # noqa: F401  (loads the CUDA runtime the library links)
    from paper_2601_19489_b200 import _lib
    if not _lib.LIB_PATH.exists():
        pytest.fail(f"{_lib.LIB_PATH} not built (run make)")
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_lib.EXPORTED_SYMBOLS)
    lib.tsr_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.tsr_version()


def test_workspace_queries_are_host_only():
    import torch  # noqa: F401
    from paper_2601_19489_b200 import _lib
    lib = _lib.load(require_cuda=False)
    assert lib.tsr_preprocess_workspace(1_000_000) > 1_000_000 // 256 * 8
    assert lib.tsr_index_workspace(1_000_000, 4_000_000) > 8 * 4 * 1_000_000


def test_product_path_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2601_19489_b200 as ts
    from paper_2601_19489_b200._lib import NativeLibraryError
    with pytest.raises((NativeLibraryError, RuntimeError, AssertionError)):
        ts.GaussianSet([[0, 0, 1.0]], [[0, 0, 0.0]], [[1, 0, 0, 0.0]], [0.0], [[0.5, 0.5, 0.5]])


def test_package_never_imports_the_oracle():
    for path in (ROOT / "paper_2601_19489_b200").rglob("*.py"):
        text = path.read_text()
        assert "from oracle" not in text and "import oracle" not in text, path
