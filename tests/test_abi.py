"""CPU checks of the drop-in boundary: the C-ABI library loads and exports every
entry point include/bzc_b200.h declares, with ctypes prototypes for each.
No compute calls (no GPU here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bzc_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bz_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared_symbols()
    for required in ("bz_compress", "bz_decompress", "bz_negate", "bz_add", "bz_mul_scalar",
                     "bz_moments", "bz_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2406_11209_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    # every declared symbol has a ctypes prototype in the binding and vice versa
    assert set(declared_symbols()) == set(_native.SIGNATURES)


def test_layout_struct_matches_header():
    from paper_2406_11209_b200 import _native

    # 4 int32 + 8 int64 + 8 int32 + 8 int64 + 2 int32 + 4 pointers
    assert ctypes.sizeof(_native.Layout) == 16 + 64 + 32 + 64 + 8 + 32
    lib = _native.load_library(require_cuda=False)
    assert lib.bz_version() >= 10000


def test_no_cpu_fallback_without_gpu():
    import torch

    from paper_2406_11209_b200 import _native

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_native.NativeUnavailable):
        _native.load_library(require_cuda=True)
