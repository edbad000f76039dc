"""Compressed-domain operations on the GPU (reference: pkg/src/bzc/ops.py).

Same names, signatures, validation and exceptions as ops.py:58-348, plus
``subtract`` (the reference composes it as add(a, negate(b)), cli.py:242).

* negate / mul_scalar / add / subtract / add_scalar run one elementwise
  kernel each and are bit-exact with the reference.
* Every scalar reduction is computed from ONE fused pass (``bz_moments``)
  that returns a partial record {n, DC means, centred DC co-moments, AC
  sums}; the closed-form epilogue below (ops.py:239-348) turns it into the
  reference's value.  Shards of a block-sharded array merge their records
  (Chan's formulas) before the epilogue -- see ``distributed.py``.
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
import torch

from . import _native
from .codec import CompressedArray, new_dc_plane, workspace
from .errors import (
    MaskExcludesMeanCoefficient,
    NegativeBaseWithFractionalWeight,
    SettingsMismatch,
    ZeroNormOperand,
)

__all__ = [
    "SsimParams",
    "negate",
    "add",
    "subtract",
    "add_scalar",
    "mul_scalar",
    "dot",
    "mean",
    "covariance",
    "variance",
    "l2_norm",
    "cosine_similarity",
    "ssim",
    "ssim_components",
    "WassersteinParams",
    "block_means",
    "approx_wasserstein",
    "subtract_l2",
    "timeseries_distances",
    "Record",
    "moments_record",
    "merge_records",
]


@dataclass(frozen=True)
class SsimParams:
    """SSIM stabilizers and weights (ops.py:58-83)."""

    luminance_stabilizer: float = 1e-4
    contrast_stabilizer: float = 9e-4
    luminance_weight: float = 1.0
    contrast_weight: float = 1.0
    structure_weight: float = 1.0

    def __post_init__(self):
        if self.luminance_stabilizer < 0 or self.contrast_stabilizer < 0:
            raise ValueError("stabilizers must be non-negative")

    @classmethod
    def for_data_range(cls, data_range: float, **weights) -> "SsimParams":
        return cls(luminance_stabilizer=(0.01 * data_range) ** 2,
                   contrast_stabilizer=(0.03 * data_range) ** 2, **weights)


# ------------------------------------------------------------- validation --
def _check_compatible(a: CompressedArray, b: CompressedArray, *, index_kind: bool = False):
    """Same checks and message format as ops.py:100-116."""
    problems = []
    if a.original_shape != b.original_shape:
        problems.append(f"shape {a.original_shape} vs {b.original_shape}")
    sa, sb = a.settings, b.settings
    if sa.block_shape != sb.block_shape:
        problems.append(f"block shape {sa.block_shape} vs {sb.block_shape}")
    if sa.mask != sb.mask:
        problems.append("pruning masks differ")
    if sa.transform is not sb.transform:
        problems.append(f"transform {sa.transform.value} vs {sb.transform.value}")
    if index_kind and sa.index_kind is not sb.index_kind:
        problems.append(f"index kind {sa.index_kind.value} vs {sb.index_kind.value}")
    if problems:
        raise SettingsMismatch("; ".join(problems))


def _require_first_coefficient(a: CompressedArray):
    if not a.settings.mask.keeps_first:
        raise MaskExcludesMeanCoefficient(
            "operation needs the first (block-mean) coefficient, but the pruning mask drops it"
        )


def _stream(a: CompressedArray) -> int:
    return _native.stream_handle(a.device)


def _derive(a: CompressedArray, maxima, indices, dc=None) -> CompressedArray:
    """Result with a's shape/settings (and a's sharding, for sharded arrays);
    `dc` is the result's DC plane when the producing kernel wrote one."""
    hook = getattr(a, "_derive", None)
    if hook is not None:
        return hook(maxima, indices, dc)
    out = CompressedArray(a.original_shape, a.settings, maxima, indices, _trusted=True, dc=dc)
    object.__setattr__(out, "_lay", a.layout())
    return out


def _new_dc(a: CompressedArray):
    return new_dc_plane(a.settings, a.maxima.shape, a.device)


# ----------------------------------------------------------- elementwise ----
@_native.on_device
def negate(a: CompressedArray) -> CompressedArray:
    """{s, N, -F}; exact (ops.py:195-197).  Maxima are shared."""
    out = torch.empty_like(a.indices)
    _native.call("bz_negate", a.settings.index_kind.code, a.indices.data_ptr(), out.data_ptr(),
                 a.indices.numel(), _stream(a))
    dc = None
    if a.dc_plane is not None:
        dc = torch.empty_like(a.dc_plane)
        _native.call("bz_negate", a.settings.index_kind.code, a.dc_plane.data_ptr(),
                     dc.data_ptr(), dc.numel(), _stream(a))
    return _derive(a, a.maxima, out, dc)


def _add(a: CompressedArray, b: CompressedArray, subtract: int) -> CompressedArray:
    _check_compatible(a, b, index_kind=True)
    out_max = torch.empty_like(a.maxima)
    out_idx = torch.empty_like(a.indices)
    dc = _new_dc(a)
    La, Lb = a.layout(), b.layout()
    bi = b.indices if b.device == a.device else b.indices.to(a.device)
    bm = b.maxima if b.device == a.device else b.maxima.to(a.device)
    _native.call("bz_add", ctypes.byref(La), ctypes.byref(Lb), a.maxima.data_ptr(),
                 a.indices.data_ptr(), bm.data_ptr(), bi.data_ptr(), subtract,
                 out_max.data_ptr(), out_idx.data_ptr(), _native.ptr(dc), _stream(a))
    return _derive(a, out_max, out_idx, dc)


@_native.on_device
def add(a: CompressedArray, b: CompressedArray) -> CompressedArray:
    """Elementwise sum with rebinning under a's kinds (ops.py:200-204); bit-exact."""
    return _add(a, b, 0)


@_native.on_device
def subtract(a: CompressedArray, b: CompressedArray) -> CompressedArray:
    """a - b == add(a, negate(b)) bit for bit, in one pass."""
    return _add(a, b, 1)


@_native.on_device
def add_scalar(a: CompressedArray, x: float) -> CompressedArray:
    """Shift each block's first coefficient by x*sqrt(prod i), rebin (ops.py:207-215)."""
    _require_first_coefficient(a)
    shift = float(x) * a.settings.block_mean_scale
    out_max = torch.empty_like(a.maxima)
    out_idx = torch.empty_like(a.indices)
    dc = _new_dc(a)
    L = a.layout()
    _native.call("bz_add_scalar", ctypes.byref(L), a.maxima.data_ptr(), a.indices.data_ptr(),
                 shift, out_max.data_ptr(), out_idx.data_ptr(), _native.ptr(dc), _stream(a))
    return _derive(a, out_max, out_idx, dc)


@_native.on_device
def mul_scalar(a: CompressedArray, x: float) -> CompressedArray:
    """N' = RN_kind(N*|x|), F' = F*sign(x) (ops.py:218-223).  x > 0 shares F."""
    x = float(x)
    out_max = torch.empty_like(a.maxima)
    out_idx = None if x > 0 else torch.empty_like(a.indices)
    dc_in = a.dc_plane
    dc_out = None if (x > 0 or dc_in is None) else torch.empty_like(dc_in)
    L = a.layout()
    _native.call("bz_mul_scalar", ctypes.byref(L), a.maxima.data_ptr(), a.indices.data_ptr(),
                 _native.ptr(dc_in), x, out_max.data_ptr(), _native.ptr(out_idx),
                 _native.ptr(dc_out), _stream(a))
    return _derive(a, out_max, a.indices if out_idx is None else out_idx,
                   dc_in if x > 0 else dc_out)


# ------------------------------------------------------------ reductions ----
class Record(NamedTuple):
    """Partial sums of one array / shard (include/bzc_b200.h, bz_moments).
    A named tuple: immutable, and built without per-field __setattr__ (this
    sits on the host path of every scalar reduction)."""

    n: float
    mean_a: float
    mean_b: float
    m_ab: float
    m_aa: float
    m_bb: float
    s_ab: float
    s_aa: float
    s_bb: float

    @classmethod
    def from_array(cls, v) -> "Record":
        return cls._make(np.asarray(v, dtype=np.float64).reshape(-1)[:9].tolist())

    def as_array(self) -> np.ndarray:
        return np.array([self.n, self.mean_a, self.mean_b, self.m_ab, self.m_aa, self.m_bb,
                         self.s_ab, self.s_aa, self.s_bb], dtype=np.float64)


def merge_records(records) -> Record:
    """Chan et al. pairwise merge, in the given (deterministic) order."""
    acc = None
    for r in records:
        if acc is None or acc.n == 0.0:
            acc = r
            continue
        if r.n == 0.0:
            continue
        n = acc.n + r.n
        da, db = r.mean_a - acc.mean_a, r.mean_b - acc.mean_b
        f = acc.n * r.n / n
        acc = Record(
            n,
            acc.mean_a + da * (r.n / n),
            acc.mean_b + db * (r.n / n),
            acc.m_ab + r.m_ab + da * db * f,
            acc.m_aa + r.m_aa + da * da * f,
            acc.m_bb + r.m_bb + db * db * f,
            acc.s_ab + r.s_ab,
            acc.s_aa + r.s_aa,
            acc.s_bb + r.s_bb,
        )
    return acc if acc is not None else Record(0, 0, 0, 0, 0, 0, 0, 0, 0)


_REDUCE_WS: dict = {}
_MOMENTS_WS_BYTES: list = []


def _reduce_workspace(dev: torch.device, La) -> torch.Tensor:
    """Zero-initialised, persistent per (device, stream) workspace: the
    reduction kernels leave their ticket counter re-armed (include/bzc_b200.h).
    Calls on one stream are ordered on the GPU, so threads sharing a stream
    may share it."""
    if not _MOMENTS_WS_BYTES:  # the size depends on no layout field
        _MOMENTS_WS_BYTES.append(int(_native.query("bz_moments_workspace", ctypes.byref(La))))
    nbytes = _MOMENTS_WS_BYTES[0]
    key = (dev.index, _native.stream_handle(dev))
    ws = _REDUCE_WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.zeros(max(nbytes, 16), dtype=torch.uint8, device=dev)
        _REDUCE_WS[key] = ws
    return ws


def moments_record(a: CompressedArray, b: CompressedArray | None = None, *,
                   dc_only: int = 0, out: torch.Tensor | None = None) -> torch.Tensor:
    """Launch the fused reduction; returns the record (16 float64) -- a new
    device tensor, or ``out`` (device memory or pinned host memory, which the
    kernel's last CTA writes directly)."""
    pair = b is not None and b is not a
    dev = a.device
    rec = out if out is not None else torch.empty(_native.RECORD_DOUBLES, dtype=torch.float64,
                                                  device=dev)
    La = a.layout()
    Lb = b.layout() if pair else La
    bm = bi = None
    if pair:
        same = b.device == dev
        bm = b.maxima if same else b.maxima.to(dev)
        bi = b.indices if same else b.indices.to(dev)
        if b.settings.index_kind is not a.settings.index_kind:
            # mixed index kinds are legal for reductions (ops.py:100-116): widen
            wide = max(a.settings.index_kind, b.settings.index_kind, key=lambda k: k.bits)
            if a.settings.index_kind is not wide:
                swapped = moments_record(b, a, dc_only=dc_only)[_SWAP_AB]
                if out is None:
                    return swapped
                out.copy_(swapped)
                return out
            conv = torch.empty(bi.shape, dtype=wide.torch_dtype, device=dev)
            _native.call("bz_convert_indices", bi.data_ptr(), b.settings.index_kind.code,
                         conv.data_ptr(), wide.code, bi.numel(), _stream(a))
            bi = conv
            from .codec import layout as _layout

            Lb = _layout(b.settings, b.original_shape, dev, index_kind=wide)
    ws = _reduce_workspace(dev, La)
    if dc_only == 1 and not pair and getattr(a, "_dc", None) is not None:
        # mean: the contiguous DC plane instead of a stride-K gather
        try:
            _native.call("bz_moments_dc", ctypes.byref(La), a.maxima.data_ptr(),
                         a._dc.data_ptr(), rec.data_ptr(), ws.data_ptr(), ws.numel(), _stream(a))
        except _native.NativeError:
            ws.zero_()
            raise
        return rec
    try:
        _native.call("bz_moments", ctypes.byref(La), ctypes.byref(Lb), a.maxima.data_ptr(),
                     a.indices.data_ptr(), bm.data_ptr() if pair else None,
                     bi.data_ptr() if pair else None, int(pair), int(dc_only), rec.data_ptr(),
                     ws.data_ptr(), ws.numel(), _stream(a))
    except _native.NativeError:
        ws.zero_()  # never leave a half-counted ticket behind a failed launch
        raise
    return rec


_SWAP_AB = [0, 2, 1, 3, 5, 4, 6, 8, 7, 9, 10, 11, 12, 13, 14, 15]
_TLS = threading.local()


def _host_record() -> torch.Tensor:
    """This thread's pinned record buffer (device-addressable under UVA):
    concurrent reductions from several threads never share one."""
    h = getattr(_TLS, "rec", None)
    if h is None:
        h = torch.empty(_native.RECORD_DOUBLES, dtype=torch.float64, pin_memory=True)
        _TLS.rec = h
        _TLS.rec_np = h.numpy()
    return h


def _host_record_np() -> np.ndarray:
    _host_record()
    return _TLS.rec_np


def record_to_host(rec: torch.Tensor) -> np.ndarray:
    """Copy a device record through this thread's pinned buffer, waiting on
    the current stream only (a pageable .cpu() copy would stall other
    streams' copies)."""
    dev = rec.device
    h = _host_record()
    h.copy_(rec, non_blocking=True)
    _native.sync_stream(dev)
    return _host_record_np().copy()


# dc_only = 2: plain sums over every kept position (no DC moments) -- all that
# dot and l2_norm need (include/bzc_b200.h, bz_moments)
_SUMS = 2


def _reduce(a, b=None, *, dc_only=False) -> Record:
    """Record of the whole array (sharded arrays merge across ranks first)."""
    hook = getattr(a, "_reduce_record", None)
    if hook is not None:
        return hook(b, dc_only)
    try:
        h, hn = _TLS.rec, _TLS.rec_np
    except AttributeError:
        h, hn = _host_record(), _host_record_np()
    pair = b is not None and b is not a
    if not pair or (b.settings.index_kind is a.settings.index_kind
                    and b._dev_index == a._dev_index):
        return _reduce_direct(a, b if pair else None, int(dc_only), h, hn)
    if pair and b.settings.index_kind is not a.settings.index_kind:
        moments_record(a, b, dc_only=dc_only, out=h)  # widened through a device copy
        _native.sync_stream(a.device)
    else:
        # the kernel's last CTA writes the record straight into this pinned
        # buffer, completion flag last: poll the flag (no stream round trip)
        hn[_native.RECORD_DOUBLES - 1] = 0.0
        moments_record(a, b, dc_only=dc_only, out=h)
        _native.call("bz_wait_record", h.data_ptr(), _stream(a))
    return Record._make(hn[:9].tolist())


def _reduce_direct(a, b, dc_only: int, h: torch.Tensor, hn: np.ndarray) -> Record:
    """The common case of _reduce -- one device, equal index kinds -- with the
    fewest host steps: one library call that launches the reduction (its last
    CTA writes the record into this thread's pinned buffer, completion flag
    last) and one that polls the flag.  Same kernels as moments_record."""
    lib = _native._lib if _native._lib is not None else _native.load_library()
    idx = a._dev_index
    stream = _native._raw_stream(idx)
    La = a.layout()
    ws = _REDUCE_WS.get((idx, stream))
    if ws is None or ws.numel() < _MOMENTS_WS_BYTES[0]:
        ws = _reduce_workspace(a.device, La)
    hp = h.data_ptr()
    hn[_native.RECORD_DOUBLES - 1] = 0.0
    if dc_only == 1 and b is None and a._dc is not None:  # mean: the DC plane
        rc = lib.bz_moments_dc(ctypes.byref(La), a.maxima.data_ptr(), a._dc.data_ptr(), hp,
                               ws.data_ptr(), ws.numel(), stream)
        name = "bz_moments_dc"
    else:
        Lb = b.layout() if b is not None else La
        rc = lib.bz_moments(ctypes.byref(La), ctypes.byref(Lb), a.maxima.data_ptr(),
                            a.indices.data_ptr(), None if b is None else b.maxima.data_ptr(),
                            None if b is None else b.indices.data_ptr(), int(b is not None),
                            dc_only, hp, ws.data_ptr(), ws.numel(), stream)
        name = "bz_moments"
    if rc:
        ws.zero_()  # never leave a half-counted ticket behind a failed launch
        raise _native.NativeError(f"{name} failed ({rc}): "
                                  f"{lib.bz_last_error().decode(errors='replace')}")
    _native.call("bz_wait_record", hp, stream)
    return Record._make(hn[:9].tolist())


def _radius(a) -> float:
    return float(a.settings.index_kind.radius)


def _global_shape(a):
    return getattr(a, "global_shape", a.original_shape)


def _global_blocks(a) -> int:
    gs = getattr(a, "global_shape", None)
    if gs is None:
        return a.block_count  # cached on the array
    return math.prod(a.settings.grid_for(gs))


def _dot_from(rec: Record, keeps_first: bool) -> float:
    dc = (rec.m_ab + rec.n * rec.mean_a * rec.mean_b) if keeps_first else 0.0
    return rec.s_ab + dc


def _sq_a(rec: Record, keeps_first: bool) -> float:
    dc = (rec.m_aa + rec.n * rec.mean_a * rec.mean_a) if keeps_first else 0.0
    return rec.s_aa + dc


def _sq_b(rec: Record, keeps_first: bool) -> float:
    dc = (rec.m_bb + rec.n * rec.mean_b * rec.mean_b) if keeps_first else 0.0
    return rec.s_bb + dc


@_native.on_device
def dot(a: CompressedArray, b: CompressedArray) -> float:
    """Dot product of the underlying arrays (ops.py:226-241)."""
    _check_compatible(a, b)
    if a.settings.mask.kept_count == 0:
        return 0.0
    rec = _reduce(a, None if a is b else b, dc_only=_SUMS)
    return _dot_from(rec, False) / (_radius(a) * _radius(b))


@_native.on_device
def l2_norm(a: CompressedArray) -> float:
    """Euclidean norm sqrt(sum (F N)^2) / r (ops.py:291-297)."""
    if a.settings.mask.kept_count == 0:
        return 0.0
    rec = _reduce(a, dc_only=_SUMS)
    return float(math.sqrt(max(_sq_a(rec, False), 0.0))) / _radius(a)


@_native.on_device
def mean(a: CompressedArray, padding_corrected: bool = False) -> float:
    """Mean from the first coefficients (ops.py:244-257)."""
    _require_first_coefficient(a)
    rec = _reduce(a, dc_only=True)
    c = a.settings.block_mean_scale
    firsts_mean = rec.mean_a / _radius(a)
    if padding_corrected:
        return float(c * (firsts_mean * rec.n) / math.prod(_global_shape(a)))
    return float(firsts_mean / c)


def _cov_from(rec_m: float, rec_s: float, a, b) -> float:
    return (rec_m + rec_s) / (_radius(a) * _radius(b)) / (_global_blocks(a) * a.settings.block_size)


@_native.on_device
def covariance(a: CompressedArray, b: CompressedArray) -> float:
    """Population covariance over the padded count (ops.py:260-283)."""
    _check_compatible(a, b)
    _require_first_coefficient(a)
    _require_first_coefficient(b)
    rec = _reduce(a, None if a is b else b)
    return _cov_from(rec.m_ab, rec.s_ab, a, b)


def variance(a: CompressedArray) -> float:
    """covariance(a, a) (ops.py:286-288)."""
    return covariance(a, a)


@_native.on_device
def cosine_similarity(a: CompressedArray, b: CompressedArray) -> float:
    """dot / (|a| |b|); ZeroNormOperand on a zero norm (ops.py:300-306).  One pass."""
    _check_compatible(a, b)
    if a.settings.mask.kept_count == 0:
        raise ZeroNormOperand("cosine similarity needs two nonzero operands")
    kf = a.settings.mask.keeps_first
    rec = _reduce(a, None if a is b else b)
    na = math.sqrt(max(_sq_a(rec, kf), 0.0)) / _radius(a)
    nb = math.sqrt(max(_sq_b(rec, kf), 0.0)) / _radius(b)
    if na == 0.0 or nb == 0.0:
        raise ZeroNormOperand("cosine similarity needs two nonzero operands")
    return (_dot_from(rec, kf) / (_radius(a) * _radius(b))) / (na * nb)


def _signed_power(base: float, weight: float, term: str) -> float:
    if base < 0 and not float(weight).is_integer():
        raise NegativeBaseWithFractionalWeight(
            f"{term} term is negative ({base!r}) with non-integer weight {weight!r}"
        )
    return float(base) ** float(weight)


@_native.on_device
def ssim_components(a: CompressedArray, b: CompressedArray,
                    params: SsimParams | None = None) -> tuple[float, float, float]:
    """Luminance, contrast, structure (ops.py:317-335), from one fused pass."""
    params = params or SsimParams()
    _check_compatible(a, b)
    _require_first_coefficient(a)
    _require_first_coefficient(b)
    rec = _reduce(a, None if a is b else b)
    c = a.settings.block_mean_scale
    mu_a = (rec.mean_a / _radius(a)) / c
    mu_b = (rec.mean_b / _radius(b)) / c
    var_a = _cov_from(rec.m_aa, rec.s_aa, a, a)
    var_b = _cov_from(rec.m_bb, rec.s_bb, b, b)
    cov = _cov_from(rec.m_ab, rec.s_ab, a, b)
    sd_a, sd_b = math.sqrt(max(var_a, 0.0)), math.sqrt(max(var_b, 0.0))
    sl, sc = params.luminance_stabilizer, params.contrast_stabilizer
    lum = (2 * mu_a * mu_b + sl) / (mu_a * mu_a + mu_b * mu_b + sl)
    con = (2 * sd_a * sd_b + sc) / (var_a + var_b + sc)
    st = (cov + sc / 2) / (sd_a * sd_b + sc / 2)
    return float(lum), float(con), float(st)


def ssim(a: CompressedArray, b: CompressedArray, params: SsimParams | None = None) -> float:
    """Weighted product of the three terms (ops.py:338-348)."""
    params = params or SsimParams()
    lum, con, st = ssim_components(a, b, params)
    return (_signed_power(lum, params.luminance_weight, "luminance")
            * _signed_power(con, params.contrast_weight, "contrast")
            * _signed_power(st, params.structure_weight, "structure"))


# ------------------------------------------------ time-series workflow --
_SL2_WS: dict = {}
_SL2_BYTES: list = []  # bz_subtract_l2_workspace(): a library constant, queried once


@_native.on_device
def _subtract_l2_sq(a: CompressedArray, b: CompressedArray, out: torch.Tensor) -> bool:
    """Squared L2 norm of subtract(a, b) into the device double ``out`` with
    the fused kernel (bz_subtract_l2); False when no fused kernel serves the
    configuration (the caller composes subtract + l2_norm, also on the GPU)."""
    _check_compatible(a, b, index_kind=True)
    dev = a.device
    key = (dev.index, _native.stream_handle(dev))
    if not _SL2_BYTES:
        _SL2_BYTES.append(int(_native.query("bz_subtract_l2_workspace")))
    nbytes = _SL2_BYTES[0]
    ws = _SL2_WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        _SL2_WS[key] = ws
    La, Lb = a.layout(), b.layout()
    bi = b.indices if b.device == dev else b.indices.to(dev)
    bm = b.maxima if b.device == dev else b.maxima.to(dev)
    rc = _native.query("bz_subtract_l2", ctypes.byref(La), ctypes.byref(Lb), a.maxima.data_ptr(),
                       a.indices.data_ptr(), bm.data_ptr(), bi.data_ptr(), out.data_ptr(),
                       ws.data_ptr(), ws.numel(), _stream(a))
    if rc == -2:  # BZ_E_UNSUPPORTED
        return False
    if rc != 0:
        ws.zero_()  # never leave a half-counted ticket behind a failed launch
        raise _native.NativeError(f"bz_subtract_l2 failed ({rc}): "
                                  f"{_native.load_library().bz_last_error().decode()}")
    return True


@_native.on_device
def subtract_l2(a: CompressedArray, b: CompressedArray) -> float:
    """l2_norm(subtract(a, b)) in one fused pass (cli.py:240-243); the same
    value as materialising the difference (rebinned under a's settings)."""
    sharded = getattr(a, "_reduce_sum", None)
    if sharded is not None:
        # each shard's fused squared norm, summed across ranks in rank order
        out = torch.empty(1, dtype=torch.float64, device=a.device)
        if not _subtract_l2_sq(a, b, out):
            return l2_norm(subtract(a, b))
        return float(math.sqrt(max(sharded(out), 0.0))) / _radius(a)
    # the kernel's last CTA stores the sum straight into this thread's pinned
    # record buffer; wait on the stream, no device scalar and no .item()
    h = _host_record()
    if not _subtract_l2_sq(a, b, h):
        return l2_norm(subtract(a, b))
    _native.sync_stream(a.device)
    return float(math.sqrt(max(float(_host_record_np()[0]), 0.0))) / _radius(a)


def timeseries_distances(snapshots, measure: str = "l2", p: float = 1.0) -> list:
    """Distances between consecutive snapshots, the reference CLI's
    ``timeseries-diff`` (cli.py:225-259): ``l2`` = l2_norm(add(s[i+1],
    negate(s[i]))) (fused, one pass per pair, one host read for all pairs);
    ``wasserstein`` = approx_wasserstein(s[i], s[i+1]) of order p."""
    snaps = list(snapshots)
    if len(snaps) < 2:
        return []
    if measure == "wasserstein":
        params = WassersteinParams(order=p)
        return [approx_wasserstein(snaps[i], snaps[i + 1], params) for i in range(len(snaps) - 1)]
    if measure != "l2":
        raise ValueError(f"unknown measure {measure!r}")
    n = len(snaps) - 1
    out = torch.empty(n, dtype=torch.float64, device=snaps[0].device)
    dists: list = [None] * n
    for i in range(n):
        if getattr(snaps[i + 1], "_reduce_record", None) is not None or \
                not _subtract_l2_sq(snaps[i + 1], snaps[i], out[i:i + 1]):
            dists[i] = l2_norm(subtract(snaps[i + 1], snaps[i]))
    host = out.cpu().numpy()
    r = _radius(snaps[0])
    return [d if d is not None else float(math.sqrt(max(float(host[i]), 0.0))) / r
            for i, d in enumerate(dists)]


# ------------------------------------------ block means / Wasserstein --
@dataclass(frozen=True)
class WassersteinParams:
    """Order and normalization tolerance for the approximate distance (ops.py:87-97)."""

    order: float = 1.0
    normalization_tolerance: float = 1e-6

    def __post_init__(self):
        if not self.order >= 1.0:
            raise ValueError(f"order must be >= 1, got {self.order}")
        if self.normalization_tolerance < 0:
            raise ValueError("normalization tolerance must be non-negative")


@_native.on_device
def block_means(a: CompressedArray) -> torch.Tensor:
    """Per-block means, flattened in row-major grid order (ops.py:355-359):
    F0 * N / r / sqrt(block size), the reference's op order; f64 on the GPU."""
    _require_first_coefficient(a)
    out = torch.empty(a.block_count, dtype=torch.float64, device=a.device)
    La = a.layout()
    if a._dc is not None:  # the DC plane: B*(idx+f) contiguous bytes, no K-strided gather
        _native.call("bz_block_means_dc", ctypes.byref(La), a.maxima.data_ptr(), a._dc.data_ptr(),
                     out.data_ptr(), _stream(a))
    else:
        _native.call("bz_block_means", ctypes.byref(La), a.maxima.data_ptr(), a.indices.data_ptr(),
                     out.data_ptr(), _stream(a))
    return out


_WS_W: dict = {}


@_native.on_device
def approx_wasserstein(a: CompressedArray, b: CompressedArray,
                       params: WassersteinParams | None = None) -> float:
    """Order-p distance between the sorted block-mean distributions
    (ops.py:362-384): block means, softmax where they do not sum to 1, device
    radix sort, (mean |d|^p)^(1/p) -- one host read of the result."""
    params = params or WassersteinParams()
    _check_compatible(a, b)
    _require_first_coefficient(a)
    _require_first_coefficient(b)
    dev = a.device
    La, Lb = a.layout(), b.layout()
    nbytes = _native.query("bz_wasserstein_workspace", ctypes.byref(La))
    key = (dev.index, _native.stream_handle(dev))
    ws = _WS_W.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        _WS_W[key] = ws
    bi = b.indices if b.device == dev else b.indices.to(dev)
    bm = b.maxima if b.device == dev else b.maxima.to(dev)
    res = torch.empty(1, dtype=torch.float64, device=dev)
    # block means from the DC planes where the producing kernels wrote them
    adc = a._dc.data_ptr() if a._dc is not None else None
    bdc = b._dc.data_ptr() if b._dc is not None and b.device == dev else None
    _native.call("bz_approx_wasserstein_dc", ctypes.byref(La), ctypes.byref(Lb),
                 a.maxima.data_ptr(), a.indices.data_ptr(), adc, bm.data_ptr(), bi.data_ptr(), bdc,
                 float(params.order), float(params.normalization_tolerance), res.data_ptr(),
                 ws.data_ptr(), ws.numel(), _stream(a))
    return float(res.item())
