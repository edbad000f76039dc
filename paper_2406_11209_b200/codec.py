"""Compression pipeline and compressed form on the GPU (reference: pkg/src/bzc/codec.py).

Names, signatures, validation and exceptions follow codec.py:67-384.  The
compressed form keeps the reference layout -- ``maxima`` shaped like the
block grid in the float kind's dtype, ``indices`` shaped ``grid + (kept,)``
in the index kind's dtype -- as CUDA tensors.  ``compress`` and
``decompress`` are single fused kernels for the common layouts
(csrc/bz_fast_*.cu) and exact per-block kernels otherwise
(csrc/bz_generic.cu).
"""

from __future__ import annotations

import ctypes
import math
import threading

import numpy as np
import torch

from . import _native
from .arrays import (
    BlockedArray,
    DenseArray,
    grid_shape,
    is_power_of_two,
    validate_shape,
)
from .errors import DimensionMismatch, IndexRangeError, LengthMismatch, NonPowerOfTwoBlock
from .kinds import FloatKind, IndexKind, kind_of_dtype, pattern_dtype, widen
from .transforms import TransformFamily, matrices_tensor, transforms_for

__all__ = [
    "PruningMask",
    "CodecSettings",
    "CompressedArray",
    "bin_coefficients",
    "prune_and_flatten",
    "unflatten",
    "compress",
    "specified_coefficients",
    "decompress",
]


class PruningMask:
    """Boolean keep/drop pattern over intrablock positions (codec.py:67-130).

    Host metadata (numpy bits); the device copy lives in the settings tables.
    """

    __slots__ = ("shape", "bits", "_key", "_kept", "_first")

    def __init__(self, shape, bits):
        shape = validate_shape(shape)
        b = np.array(bits, dtype=bool, copy=True, order="C")
        if b.shape != shape:
            raise DimensionMismatch(f"mask bits shaped {b.shape} do not match mask shape {shape}")
        b.flags.writeable = False
        object.__setattr__(self, "shape", shape)
        object.__setattr__(self, "bits", b)
        object.__setattr__(self, "_key", (shape, b.tobytes()))
        # immutable: the scalars every operator asks for are computed once
        object.__setattr__(self, "_kept", int(b.sum()))
        object.__setattr__(self, "_first", bool(b.flat[0]) if b.size else False)

    def __setattr__(self, name, value):
        raise AttributeError("PruningMask is immutable")

    @property
    def kept_count(self) -> int:
        return self._kept

    @property
    def flat_kept(self) -> np.ndarray:
        return np.flatnonzero(self.bits.ravel())

    @property
    def keeps_first(self) -> bool:
        return self._first

    @classmethod
    def full(cls, shape) -> "PruningMask":
        shape = validate_shape(shape)
        return cls(shape, np.ones(shape, dtype=bool))

    @classmethod
    def first_k(cls, shape, k: int) -> "PruningMask":
        shape = validate_shape(shape)
        n = int(np.prod(shape))
        if not 0 <= k <= n:
            raise ValueError(f"kept count {k} outside [0, {n}]")
        bits = np.zeros(n, dtype=bool)
        bits[:k] = True
        return cls(shape, bits.reshape(shape))

    @classmethod
    def from_bits(cls, shape, bits) -> "PruningMask":
        shape = validate_shape(shape)
        flat = np.asarray(bits, dtype=bool).ravel()
        if flat.size != int(np.prod(shape)):
            raise LengthMismatch(f"{flat.size} mask bits for block shape {shape}")
        return cls(shape, flat.reshape(shape))

    def __eq__(self, other):
        if not isinstance(other, PruningMask):
            return NotImplemented
        return self._key == other._key

    def __hash__(self):
        return hash(self._key)


class CodecSettings:
    """Block shape, float kind, index kind, transform, mask (codec.py:133-179)."""

    __slots__ = ("block_shape", "float_kind", "index_kind", "transform", "mask", "_bsize")

    def __init__(self, block_shape, float_kind: FloatKind = FloatKind.F32,
                 index_kind: IndexKind = IndexKind.I16,
                 transform: TransformFamily = TransformFamily.DCT,
                 mask: PruningMask | None = None):
        bshape = validate_shape(block_shape)
        if not all(is_power_of_two(b) for b in bshape):
            raise NonPowerOfTwoBlock(f"block extents must be powers of two, got {bshape}")
        mask = mask if mask is not None else PruningMask.full(bshape)
        if mask.shape != bshape:
            raise DimensionMismatch(f"mask shaped {mask.shape} does not match block shape {bshape}")
        for k, v in (("block_shape", bshape), ("float_kind", float_kind),
                     ("index_kind", index_kind), ("transform", transform), ("mask", mask)):
            object.__setattr__(self, k, v)
        object.__setattr__(self, "_bsize", math.prod(bshape))

    def __setattr__(self, name, value):
        raise AttributeError("CodecSettings is immutable")

    def _key(self):
        return (self.block_shape, self.float_kind, self.index_kind, self.transform, self.mask)

    def __eq__(self, other):
        if not isinstance(other, CodecSettings):
            return NotImplemented
        return self._key() == other._key()

    def __hash__(self):
        return hash(self._key())

    def __repr__(self):
        return (f"CodecSettings(block_shape={self.block_shape}, float_kind={self.float_kind.value}, "
                f"index_kind={self.index_kind.value}, transform={self.transform.value}, "
                f"kept={self.mask.kept_count})")

    @property
    def ndim(self) -> int:
        return len(self.block_shape)

    @property
    def block_size(self) -> int:
        return self._bsize

    @property
    def block_mean_scale(self) -> float:
        return math.sqrt(self._bsize)  # correctly rounded, as np.sqrt

    def grid_for(self, shape) -> tuple[int, ...]:
        shape = validate_shape(shape)
        if len(shape) != self.ndim:
            raise DimensionMismatch(
                f"settings are {self.ndim}-dimensional, array shape {shape} is not"
            )
        return grid_shape(shape, self.block_shape)

    def matrices(self):
        return transforms_for(self.block_shape, self.transform)


# ------------------------------------------------------------ device tables --
_TABLES: dict = {}
_TABLES_LOCK = threading.Lock()


def _tables(settings: CodecSettings, device: torch.device):
    """(kept_pos, rank, matrices) device tensors for `settings`, cached."""
    key = (settings, device.index)
    t = _TABLES.get(key)
    if t is None:
        with _TABLES_LOCK:
            t = _TABLES.get(key)
            if t is None:
                kept = settings.mask.flat_kept.astype(np.int32)
                rank = np.full(settings.block_size, -1, dtype=np.int32)
                rank[kept] = np.arange(kept.size, dtype=np.int32)
                host = np.ascontiguousarray(
                    np.concatenate([m.entries.reshape(-1) for m in settings.matrices()]))
                t = (
                    torch.from_numpy(kept if kept.size else np.zeros(1, np.int32)).to(device),
                    torch.from_numpy(rank).to(device),
                    matrices_tensor(settings.matrices(), device),
                    host,
                )
                _TABLES[key] = t
    return t


def layout(settings: CodecSettings, shape, device: torch.device, *,
           index_kind: IndexKind | None = None) -> _native.Layout:
    """The C-ABI descriptor of an array of `shape` compressed with `settings`."""
    kept_pos, rank, mats, host = _tables(settings, device)
    L = _native.Layout()
    L.ndim = settings.ndim
    L.float_kind = settings.float_kind.code
    L.index_kind = (index_kind or settings.index_kind).code
    L.transform = settings.transform.code
    for a, (s, b) in enumerate(zip(shape, settings.block_shape)):
        L.shape[a] = int(s)
        L.block[a] = int(b)
        L.grid[a] = -(-int(s) // int(b))
    L.kept = settings.mask.kept_count
    L.keeps_first = int(settings.mask.keeps_first)
    L.kept_pos = kept_pos.data_ptr()
    L.rank = rank.data_ptr()
    L.matrices = mats.data_ptr()
    L.matrices_host = host.ctypes.data
    return L


def workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)


def _device():
    return torch.device("cuda", torch.cuda.current_device())


# ---------------------------------------------------------- compressed form --
class CompressedArray:
    """{original_shape, settings, maxima, indices} (codec.py:182-250).

    Equality is bit-exact (maxima compared as raw bit patterns).  Tensors
    are treated as immutable; operations may return arrays that share an
    operand's unchanged maxima or indices (negate, mul_scalar).
    """

    __slots__ = ("original_shape", "settings", "maxima", "indices", "_lay", "_dc", "_dev", "_nb",
                 "_didx")

    def __init__(self, original_shape, settings: CodecSettings, maxima, indices, *,
                 _trusted: bool = False, dc=None):
        shape = validate_shape(original_shape)
        grid = settings.grid_for(shape)
        if _trusted:
            m, idx = maxima, indices
        else:
            dev = maxima.device if isinstance(maxima, torch.Tensor) and maxima.is_cuda else _device()
            m = _to_float_storage(maxima, settings.float_kind, dev)
            idx = _to_index_storage(indices, settings.index_kind, dev)
        if tuple(m.shape) != grid:
            raise DimensionMismatch(f"maxima shaped {tuple(m.shape)}, expected block grid {grid}")
        expected = grid + (settings.mask.kept_count,)
        if tuple(idx.shape) != expected:
            raise DimensionMismatch(f"indices shaped {tuple(idx.shape)}, expected {expected}")
        if not _trusted:
            r = settings.index_kind.radius
            if idx.numel() and int(idx.min()) < -r:
                raise IndexRangeError(f"bin index {int(idx.min())} below -{r}")
        for k, v in (("original_shape", shape), ("settings", settings), ("maxima", m),
                     ("indices", idx)):
            object.__setattr__(self, k, v)
        # DC plane: the first coefficient of every block, contiguous (written by
        # the producing kernel; a cache of indices[..., 0], not part of equality)
        object.__setattr__(self, "_dc", dc if _trusted else None)

    def __setattr__(self, name, value):
        raise AttributeError("CompressedArray is immutable")

    @property
    def block_grid(self) -> tuple[int, ...]:
        return self.settings.grid_for(self.original_shape)

    @property
    def block_count(self) -> int:
        nb = getattr(self, "_nb", None)  # immutable: computed once
        if nb is None:
            nb = math.prod(self.block_grid)
            object.__setattr__(self, "_nb", nb)
        return nb

    @property
    def device(self) -> torch.device:
        dev = getattr(self, "_dev", None)
        if dev is None:
            dev = self.indices.device
            object.__setattr__(self, "_dev", dev)
        return dev

    @property
    def _dev_index(self):
        """CUDA device index (None for CPU tensors), cached."""
        i = getattr(self, "_didx", None)
        if i is None:
            d = self.device
            i = d.index if d.type == "cuda" else -1
            object.__setattr__(self, "_didx", i)
        return None if i < 0 else i

    @property
    def dc_plane(self) -> torch.Tensor | None:
        """indices[..., 0] as a contiguous grid-shaped tensor when the producing
        kernel wrote it (compress / add / scalar ops), else None."""
        return self._dc

    def maxima_f64(self) -> torch.Tensor:
        return widen(self.maxima)

    def maxima_bits(self) -> torch.Tensor:
        return self.maxima.view(pattern_dtype(self.settings.float_kind))

    def layout(self) -> _native.Layout:
        """The C-ABI descriptor, built once per array (the array is immutable)."""
        L = getattr(self, "_lay", None)
        if L is None:
            L = layout(self.settings, self.original_shape, self.device)
            object.__setattr__(self, "_lay", L)
        return L

    def __eq__(self, other):
        if not isinstance(other, CompressedArray):
            return NotImplemented
        return (
            self.original_shape == other.original_shape
            and self.settings == other.settings
            and torch.equal(self.maxima_bits(), other.maxima_bits().to(self.device))
            and torch.equal(self.indices, other.indices.to(self.device))
        )

    __hash__ = object.__hash__

    def __repr__(self):
        return (f"CompressedArray(shape={self.original_shape}, {self.settings!r}, "
                f"device={self.device})")


def _to_float_storage(values, kind: FloatKind, device) -> torch.Tensor:
    if isinstance(values, torch.Tensor) and values.dtype == kind.torch_dtype:
        return values.to(device).clone().contiguous()
    from .kinds import to_storage

    return to_storage(values if not isinstance(values, torch.Tensor) else values.to(device), kind)


def _to_index_storage(values, kind: IndexKind, device) -> torch.Tensor:
    if isinstance(values, torch.Tensor):
        return values.to(device=device, dtype=kind.torch_dtype).clone().contiguous()
    arr = np.ascontiguousarray(np.asarray(values).astype(kind.dtype))
    return torch.from_numpy(arr).to(device)


# ------------------------------------------------------------------ codec ----
@_native.on_device
def compress(a: DenseArray, settings: CodecSettings) -> CompressedArray:
    """convert -> block -> transform -> bin -> prune (codec.py:321-334), fused."""
    if a.ndim != settings.ndim:
        raise DimensionMismatch(
            f"settings are {settings.ndim}-dimensional, array is {a.ndim}-dimensional"
        )
    dev = a.values.device
    grid = settings.grid_for(a.shape)
    maxima = torch.empty(grid, dtype=settings.float_kind.torch_dtype, device=dev)
    indices = torch.empty(grid + (settings.mask.kept_count,), dtype=settings.index_kind.torch_dtype,
                          device=dev)
    dc = new_dc_plane(settings, grid, dev)
    L = layout(settings, a.shape, dev)
    ws = workspace(_native.query("bz_compress_workspace", ctypes.byref(L)), dev)
    _native.call("bz_compress", ctypes.byref(L), a.values.data_ptr(), a.kind.code,
                 maxima.data_ptr(), indices.data_ptr(), _native.ptr(dc), ws.data_ptr(),
                 ws.numel(), _native.stream_handle(dev))
    out = CompressedArray(a.shape, settings, maxima, indices, _trusted=True, dc=dc)
    object.__setattr__(out, "_lay", L)
    return out


def new_dc_plane(settings: CodecSettings, grid, device) -> torch.Tensor | None:
    """Storage for a result's DC plane (None when the mask drops position 0)."""
    if not settings.mask.keeps_first or settings.mask.kept_count == 0:
        return None
    return torch.empty(grid, dtype=settings.index_kind.torch_dtype, device=device)


@_native.on_device
def decompress(a: CompressedArray, out_kind: FloatKind = FloatKind.F64) -> DenseArray:
    """Inverse transform, *N, /r, merge, crop (codec.py:364-384), fused.

    Output values are float64 as in the reference; ``out_kind`` (extension)
    rounds the same float64 results once into a narrower kind, halving or
    quartering the bytes written.
    """
    dev = a.device
    out = torch.empty(a.original_shape, dtype=out_kind.torch_dtype, device=dev)
    L = a.layout()
    ws = workspace(_native.query("bz_decompress_workspace", ctypes.byref(L)), dev)
    _native.call("bz_decompress", ctypes.byref(L), a.maxima.data_ptr(), a.indices.data_ptr(),
                 out.data_ptr(), out_kind.code, ws.data_ptr(), ws.numel(),
                 _native.stream_handle(dev))
    return DenseArray(a.original_shape, out_kind, out, _trusted=True)


def _mask_layout(mask: PruningMask, grid, index_kind: IndexKind, device,
                 float_kind: FloatKind = FloatKind.F64) -> _native.Layout:
    settings = CodecSettings(mask.shape, float_kind, index_kind, TransformFamily.DCT, mask)
    shape = tuple(g * b for g, b in zip(grid, mask.shape))
    return layout(settings, shape, device)


def bin_coefficients(c: BlockedArray, index_kind: IndexKind,
                     float_kind: FloatKind = FloatKind.F64):
    """(maxima, indices) of coefficient blocks (codec.py:253-278).

    maxima: block grid in float_kind's dtype; indices: grid + block shape.
    """
    dev = c.blocks.device
    maxima = torch.empty(c.block_grid, dtype=float_kind.torch_dtype, device=dev)
    full = torch.empty(c.block_grid + c.block_shape, dtype=index_kind.torch_dtype, device=dev)
    L = _mask_layout(PruningMask.full(c.block_shape), c.block_grid, index_kind, dev, float_kind)
    _native.call("bz_bin", ctypes.byref(L), c.blocks.contiguous().data_ptr(), maxima.data_ptr(),
                 full.data_ptr(), _native.stream_handle(dev))
    return maxima, full


def _index_kind_of(t: torch.Tensor) -> IndexKind:
    for k in IndexKind:
        if k.torch_dtype == t.dtype:
            return k
    raise TypeError(f"indices must be an integer tensor, got {t.dtype}")


def prune_and_flatten(indices, mask: PruningMask) -> torch.Tensor:
    """Kept positions, row-major, shaped grid + (kept,) (codec.py:281-297)."""
    t = indices if isinstance(indices, torch.Tensor) else _to_index_storage(
        indices, IndexKind.I64 if np.asarray(indices).dtype == np.int64 else
        {1: IndexKind.I8, 2: IndexKind.I16, 4: IndexKind.I32}.get(np.asarray(indices).dtype.itemsize, IndexKind.I64),
        _device())
    d = len(mask.shape)
    if tuple(t.shape[-d:]) != mask.shape:
        raise DimensionMismatch(f"index blocks shaped {tuple(t.shape[-d:])}, mask {mask.shape}")
    grid = tuple(t.shape[:-d])
    out = torch.empty(grid + (mask.kept_count,), dtype=t.dtype, device=t.device)
    if out.numel() and grid:
        L = _mask_layout(mask, grid, _index_kind_of(t), t.device)
        _native.call("bz_prune", ctypes.byref(L), t.contiguous().data_ptr(), out.data_ptr(),
                     _native.stream_handle(t.device))
    return out


def unflatten(flat, mask: PruningMask) -> torch.Tensor:
    """Inverse of prune_and_flatten, zeros at dropped positions (codec.py:300-318)."""
    t = flat if isinstance(flat, torch.Tensor) else _to_index_storage(
        flat, {1: IndexKind.I8, 2: IndexKind.I16, 4: IndexKind.I32, 8: IndexKind.I64}[np.asarray(flat).dtype.itemsize],
        _device())
    if t.shape[-1] != mask.kept_count:
        raise LengthMismatch(f"{t.shape[-1]} indices per block, mask keeps {mask.kept_count}")
    grid = tuple(t.shape[:-1])
    out = torch.empty(grid + mask.shape, dtype=t.dtype, device=t.device)
    if out.numel() and grid:
        L = _mask_layout(mask, grid, _index_kind_of(t), t.device)
        _native.call("bz_unflatten", ctypes.byref(L), t.contiguous().data_ptr(), out.data_ptr(),
                     _native.stream_handle(t.device))
    return out


@_native.on_device
def specified_coefficients(a: CompressedArray) -> BlockedArray:
    """(F * N) / r per kept position, zeros elsewhere (codec.py:337-361)."""
    out = torch.empty(a.block_grid + a.settings.block_shape, dtype=torch.float64, device=a.device)
    L = a.layout()
    _native.call("bz_specified", ctypes.byref(L), a.maxima.data_ptr(), a.indices.data_ptr(),
                 out.data_ptr(), _native.stream_handle(a.device))
    return BlockedArray(a.block_grid, a.settings.block_shape, a.original_shape,
                        a.settings.float_kind, out, _trusted=True)


def is_fast_path(settings: CodecSettings, shape) -> bool:
    """True when compress dispatches to the fused single-pass kernel."""
    L = layout(settings, shape, _device())
    return bool(_native.query("bz_fast_path", ctypes.byref(L)))
