"""ctypes binding of the sm_100a C-ABI library (include/bzc_b200.h).

The library is built in-tree (``paper_2406_11209_b200/libbzc_b200.so``, see
``__graft_entry__.build``).  There is no CPU fallback: if the library or a
CUDA device is missing, every compute entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import functools
import os
import threading

import torch

from .errors import BzcError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BZC_B200_LIB", os.path.join(_HERE, "libbzc_b200.so"))

MAX_DIMS = 8
RECORD_DOUBLES = 16


class NativeUnavailable(BzcError):
    """The CUDA library or a CUDA device is not available (no CPU fallback)."""


class NativeError(BzcError):
    """A kernel launch or CUDA call failed inside the native library."""


class Layout(ctypes.Structure):
    """Mirror of ``struct bz_layout`` (include/bzc_b200.h)."""

    _fields_ = [
        ("ndim", ctypes.c_int32),
        ("float_kind", ctypes.c_int32),
        ("index_kind", ctypes.c_int32),
        ("transform", ctypes.c_int32),
        ("shape", ctypes.c_int64 * MAX_DIMS),
        ("block", ctypes.c_int32 * MAX_DIMS),
        ("grid", ctypes.c_int64 * MAX_DIMS),
        ("kept", ctypes.c_int32),
        ("keeps_first", ctypes.c_int32),
        ("kept_pos", ctypes.c_void_p),
        ("rank", ctypes.c_void_p),
        ("matrices", ctypes.c_void_p),
        ("matrices_host", ctypes.c_void_p),
    ]


_P = ctypes.c_void_p
_L = ctypes.POINTER(Layout)
_I = ctypes.c_int
_I64 = ctypes.c_int64
_SZ = ctypes.c_size_t
_D = ctypes.c_double

# name -> (restype, argtypes); every symbol include/bzc_b200.h declares
SIGNATURES = {
    "bz_version": (_I, []),
    "bz_last_error": (ctypes.c_char_p, []),
    "bz_launch_count": (ctypes.c_longlong, []),
    "bz_fast_path": (_I, [_L]),
    "bz_stream_sync": (_I, [_P]),
    "bz_wait_record": (_I, [_P, _P]),
    "bz_compress_workspace": (_SZ, [_L]),
    "bz_compress": (_I, [_L, _P, _I, _P, _P, _P, _P, _SZ, _P]),
    "bz_decompress_workspace": (_SZ, [_L]),
    "bz_decompress": (_I, [_L, _P, _P, _P, _I, _P, _SZ, _P]),
    "bz_negate": (_I, [_I, _P, _P, _I64, _P]),
    "bz_mul_scalar": (_I, [_L, _P, _P, _P, _D, _P, _P, _P, _P]),
    "bz_add": (_I, [_L, _L, _P, _P, _P, _P, _I, _P, _P, _P, _P]),
    "bz_add_scalar": (_I, [_L, _P, _P, _D, _P, _P, _P, _P]),
    "bz_extract_dc": (_I, [_L, _P, _P, _P]),
    "bz_moments_workspace": (_SZ, [_L]),
    "bz_moments": (_I, [_L, _L, _P, _P, _P, _P, _I, _I, _P, _P, _SZ, _P]),
    "bz_moments_dc": (_I, [_L, _P, _P, _P, _P, _SZ, _P]),
    "bz_round_to_kind": (_I, [_P, _I, _P, _I, _I64, _P, _P]),
    "bz_gradient": (_I, [_I, ctypes.POINTER(ctypes.c_int64), _I, _P, _P]),
    "bz_block": (_I, [_L, _P, _I, _P, _P]),
    "bz_unblock": (_I, [_L, _P, _P, _I, _P]),
    "bz_transform": (_I, [_L, _P, _P, _I, _P, _SZ, _P]),
    "bz_bin": (_I, [_L, _P, _P, _P, _P]),
    "bz_prune": (_I, [_L, _P, _P, _P]),
    "bz_unflatten": (_I, [_L, _P, _P, _P]),
    "bz_specified": (_I, [_L, _P, _P, _P, _P]),
    "bz_convert_indices": (_I, [_P, _I, _P, _I, _I64, _P]),
    "bz_fill_random": (_I, [_P, _I, _I64, _I64, ctypes.c_uint64, _I, _P]),
    "bz_block_means": (_I, [_L, _P, _P, _P, _P]),
    "bz_block_means_dc": (_I, [_L, _P, _P, _P, _P]),
    "bz_wasserstein_workspace": (_SZ, [_L]),
    "bz_approx_wasserstein": (_I, [_L, _L, _P, _P, _P, _P, _D, _D, _P, _P, _SZ, _P]),
    "bz_approx_wasserstein_dc": (_I, [_L, _L, _P, _P, _P, _P, _P, _P, _D, _D, _P, _P, _SZ, _P]),
    "bz_subtract_l2_workspace": (_SZ, []),
    "bz_subtract_l2": (_I, [_L, _L, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "bz_error_bounds": (_I, [_L, _P, _P, _P, _P, _P, _P, _P]),
    "bz_block_diff": (_I, [_I64, _I, _P, _P, _P, _P, _P]),
    "bz_stream_pack": (_I, [_P, _I64, _P, _I64, _I64, ctypes.c_uint32, _P, _I64, _P]),
    "bz_stream_unpack": (_I, [_P, _I64, _I64, _P, _I64, _P, _I64, _P]),
}

_lib = None
_lock = threading.Lock()


def load_library(require_cuda: bool = True):
    """Load (once) and return the ctypes library; raise if unusable."""
    global _lib
    if require_cuda and not torch.cuda.is_available():
        raise NativeUnavailable(
            "paper_2406_11209_b200 needs a CUDA device (B200, sm_100a); no CPU fallback"
        )
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise NativeUnavailable(
                        f"native library {LIB_PATH} is missing; run __graft_entry__.build()"
                    )
                lib = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = lib
    return _lib


_raw_stream = torch._C._cuda_getCurrentRawStream


def stream_handle(device=None) -> int:
    """The current stream's cudaStream_t for `device` (an int; no Stream
    object is built, which keeps per-call host overhead low)."""
    if device is None:
        return _raw_stream(_current_device())
    idx = device.index if isinstance(device, torch.device) else device
    return _raw_stream(_current_device() if idx is None else int(idx))


def sync_stream(device=None) -> None:
    """Wait for the current stream of `device` (only that stream), through
    the library (cudaStreamSynchronize with the GIL released) -- a fraction
    of the host cost of building a torch Stream object and syncing it."""
    call("bz_stream_sync", stream_handle(device))


def call(name: str, *args) -> int:
    """Call a status-returning entry point; raise NativeError on failure."""
    lib = _lib if _lib is not None else load_library()  # loaded once: no per-call CUDA query
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.bz_last_error().decode(errors="replace")
        raise NativeError(f"{name} failed ({rc}): {msg}")
    return rc


def query(name: str, *args):
    return getattr(load_library(), name)(*args)


def _device_of(x):
    dev = getattr(x, "device", None)
    if dev is None:
        vals = getattr(x, "values", None)
        dev = getattr(vals, "device", None)
    return dev


_current_device = torch._C._cuda_getDevice


def on_device(fn):
    """Run a public operator with its first operand's GPU current, so the
    library's launches, occupancy queries and attribute calls (which act on
    the current device) target the device that holds the data."""

    @functools.wraps(fn)
    def wrapper(a, *args, **kwargs):
        idx = getattr(a, "_dev_index", None)  # CompressedArray caches it
        if idx is None:
            dev = _device_of(a)
            idx = dev.index if dev is not None and dev.type == "cuda" else None
        if idx is not None and idx != _current_device():
            with torch.cuda.device(idx):
                return fn(a, *args, **kwargs)
        return fn(a, *args, **kwargs)

    return wrapper


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr()
