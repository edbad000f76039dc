"""Element kinds (reference: pkg/src/bzc/kinds.py).

``FloatKind`` / ``IndexKind`` keep the reference's values, properties and
2-bit codes (kinds.py:30-183).  Storage is a torch dtype on the GPU:
bf16 -> torch.bfloat16, f16 -> torch.float16, f32 -> torch.float32,
f64 -> torch.float64; index kinds map to torch.int8 .. torch.int64.
``round_to_kind`` runs the IEEE round-to-nearest-even kernel on the device
(bz_round_to_kind, same algorithm as kinds.py:186-206).
"""

from __future__ import annotations

import enum
import math

import numpy as np
import torch

__all__ = [
    "FloatKind",
    "IndexKind",
    "round_to_kind",
    "storage_dtype",
    "to_storage",
    "from_storage",
    "pattern_dtype",
]


class FloatKind(enum.Enum):
    """Floating-point element format (kinds.py:30-81)."""

    BF16 = "bf16"
    F16 = "f16"
    F32 = "f32"
    F64 = "f64"

    @property
    def bits(self) -> int:
        return _FLOAT_INFO[self][0]

    @property
    def significand_bits(self) -> int:
        return _FLOAT_INFO[self][1]

    @property
    def exponent_bits(self) -> int:
        return _FLOAT_INFO[self][2]

    @property
    def precision(self) -> int:
        return self.significand_bits + 1

    @property
    def max_exponent(self) -> int:
        return 2 ** (self.exponent_bits - 1) - 1

    @property
    def min_exponent(self) -> int:
        return 1 - self.max_exponent

    @property
    def max_finite(self) -> float:
        return float((2.0 - 2.0 ** (1 - self.precision)) * 2.0 ** self.max_exponent)

    @property
    def code(self) -> int:
        return _FLOAT_CODE[self]

    @property
    def torch_dtype(self) -> torch.dtype:
        return _TORCH_FLOAT[self]

    @property
    def itemsize(self) -> int:
        return self.bits // 8

    @classmethod
    def from_code(cls, code: int) -> "FloatKind":
        return _FLOAT_BY_CODE[code]

    @classmethod
    def parse(cls, name: str) -> "FloatKind":
        return cls(name.strip().lower())


_FLOAT_INFO = {
    FloatKind.BF16: (16, 7, 8),
    FloatKind.F16: (16, 10, 5),
    FloatKind.F32: (32, 23, 8),
    FloatKind.F64: (64, 52, 11),
}
_FLOAT_CODE = {FloatKind.BF16: 0, FloatKind.F16: 1, FloatKind.F32: 2, FloatKind.F64: 3}
_FLOAT_BY_CODE = {v: k for k, v in _FLOAT_CODE.items()}
_TORCH_FLOAT = {
    FloatKind.BF16: torch.bfloat16,
    FloatKind.F16: torch.float16,
    FloatKind.F32: torch.float32,
    FloatKind.F64: torch.float64,
}
_KIND_OF_TORCH = {v: k for k, v in _TORCH_FLOAT.items()}
_PATTERN = {
    FloatKind.BF16: torch.int16,
    FloatKind.F16: torch.int16,
    FloatKind.F32: torch.int32,
    FloatKind.F64: torch.int64,
}


class IndexKind(enum.Enum):
    """Signed integer bin-index format (kinds.py:115-160)."""

    I8 = "i8"
    I16 = "i16"
    I32 = "i32"
    I64 = "i64"

    @property
    def bits(self) -> int:
        return _INDEX_BITS[self]

    @property
    def radius(self) -> int:
        """r = 2**(b-1) - 1."""
        return 2 ** (self.bits - 1) - 1

    @property
    def dtype(self) -> np.dtype:
        """numpy dtype of the index kind (host views, as in the reference)."""
        return np.dtype(f"int{self.bits}")

    @property
    def torch_dtype(self) -> torch.dtype:
        return _TORCH_INDEX[self]

    @property
    def itemsize(self) -> int:
        return self.bits // 8

    @property
    def clamp_bound(self) -> float:
        """Largest float64 not above the radius (2**63-1024 for I64)."""
        r = float(self.radius)
        if r > self.radius:
            r = math.nextafter(r, 0.0)
        return float(r)

    @property
    def code(self) -> int:
        return _INDEX_CODE[self]

    @classmethod
    def from_code(cls, code: int) -> "IndexKind":
        return _INDEX_BY_CODE[code]

    @classmethod
    def parse(cls, name: str) -> "IndexKind":
        return cls(name.strip().lower())


_INDEX_BITS = {IndexKind.I8: 8, IndexKind.I16: 16, IndexKind.I32: 32, IndexKind.I64: 64}
_INDEX_CODE = {IndexKind.I8: 0, IndexKind.I16: 1, IndexKind.I32: 2, IndexKind.I64: 3}
_INDEX_BY_CODE = {v: k for k, v in _INDEX_CODE.items()}
_TORCH_INDEX = {
    IndexKind.I8: torch.int8,
    IndexKind.I16: torch.int16,
    IndexKind.I32: torch.int32,
    IndexKind.I64: torch.int64,
}


def kind_of_dtype(dtype: torch.dtype) -> FloatKind | None:
    return _KIND_OF_TORCH.get(dtype)


def storage_dtype(kind: FloatKind) -> torch.dtype:
    """Native torch dtype used to store values of `kind`."""
    return kind.torch_dtype


def pattern_dtype(kind: FloatKind) -> torch.dtype:
    """Integer dtype of the same width, for raw bit patterns."""
    return _PATTERN[kind]


def as_device_tensor(values, device=None) -> torch.Tensor:
    """Any array-like -> contiguous CUDA tensor (float kinds kept, others -> f64)."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    if isinstance(values, torch.Tensor):
        t = values
        if t.dtype not in _KIND_OF_TORCH:
            t = t.to(torch.float64)
        # pinned host memory: asynchronous H2D on the current stream
        return t.to(dev, non_blocking=(not t.is_cuda and t.is_pinned())).contiguous()
    arr = np.asarray(values)
    if arr.dtype == np.float32:
        t = torch.from_numpy(np.ascontiguousarray(arr))
    elif arr.dtype == np.float16:
        t = torch.from_numpy(np.ascontiguousarray(arr))
    elif arr.dtype.name == "bfloat16":
        t = torch.from_numpy(np.ascontiguousarray(arr).view(np.int16)).view(torch.bfloat16)
    else:
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64))
    return t.to(dev, non_blocking=False).contiguous()


def round_to_kind(values, kind: FloatKind) -> torch.Tensor:
    """IEEE round-to-nearest-even into `kind`, returned as a float64 CUDA tensor.

    Same contract as kinds.py:186-206 (ties to even, overflow -> signed inf,
    NaN / inf / signed zero pass through), computed by the device kernel.
    """
    from . import _native

    src = as_device_tensor(values)
    out = torch.empty(src.shape, dtype=torch.float64, device=src.device)
    in_kind = kind_of_dtype(src.dtype)
    # round into kind, widen back: two passes through the same kernel
    tmp = torch.empty(src.shape, dtype=kind.torch_dtype, device=src.device)
    n = src.numel()
    s = _native.stream_handle(src.device)
    _native.call("bz_round_to_kind", src.data_ptr(), in_kind.code, tmp.data_ptr(), kind.code, n, None, s)
    _native.call("bz_round_to_kind", tmp.data_ptr(), kind.code, out.data_ptr(), FloatKind.F64.code, n, None, s)
    return out


def to_storage(values, kind: FloatKind) -> torch.Tensor:
    """Round into `kind` and store in its native dtype (CUDA tensor)."""
    from . import _native

    src = as_device_tensor(values)
    out = torch.empty(src.shape, dtype=kind.torch_dtype, device=src.device)
    _native.call("bz_round_to_kind", src.data_ptr(), kind_of_dtype(src.dtype).code, out.data_ptr(),
                 kind.code, src.numel(), None, _native.stream_handle(src.device))
    return out


def from_storage(values: torch.Tensor) -> torch.Tensor:
    """Widen stored values to float64 (exact)."""
    return widen(values)


def widen(values: torch.Tensor) -> torch.Tensor:
    from . import _native

    values = values.contiguous()
    kind = kind_of_dtype(values.dtype)
    out = torch.empty(values.shape, dtype=torch.float64, device=values.device)
    if values.numel():
        _native.call("bz_round_to_kind", values.data_ptr(), kind.code, out.data_ptr(),
                     FloatKind.F64.code, values.numel(), None, _native.stream_handle(values.device))
    return out
