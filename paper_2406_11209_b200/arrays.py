"""Dense and blocked arrays on the GPU (reference: pkg/src/bzc/arrays.py).

``DenseArray`` keeps the reference's fields ``(shape, kind, values)`` and its
contract that every value is exactly representable in ``kind``
(arrays.py:65-101); ``values`` is a CUDA tensor in the kind's native dtype
(bf16/f16/f32/f64), so an F32 array occupies 4 bytes per element in HBM
instead of the reference's 8.  ``BlockedArray`` holds float64 blocks shaped
``grid + block`` (arrays.py:104-144).  Blocking, unblocking, precision
conversion and the gradient generator run as CUDA kernels.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .errors import DegenerateShape, DimensionMismatch, NonPowerOfTwoBlock
from .kinds import FloatKind, as_device_tensor, kind_of_dtype

__all__ = [
    "DenseArray",
    "BlockedArray",
    "convert_precision",
    "block",
    "unblock",
    "gradient_array",
    "validate_shape",
    "is_power_of_two",
    "grid_shape",
]


def validate_shape(dims) -> tuple[int, ...]:
    """Tuple of positive ints or DegenerateShape (arrays.py:32-39)."""
    shape = tuple(int(d) for d in dims)
    if len(shape) < 1:
        raise DegenerateShape("shape must have at least one axis")
    if any(d < 1 for d in shape):
        raise DegenerateShape(f"every extent must be >= 1, got {shape}")
    return shape


def is_power_of_two(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


def grid_shape(shape, block_shape) -> tuple[int, ...]:
    """ceil(shape / block) per axis (arrays.py:46-48)."""
    return tuple(-(-int(s) // int(b)) for s, b in zip(shape, block_shape))


def _stream(t: torch.Tensor) -> int:
    return _native.stream_handle(t.device)


def _round_into(src: torch.Tensor, kind: FloatKind, check: bool) -> torch.Tensor:
    """Device round-to-kind copy; with check=True raise if any value changed."""
    out = torch.empty(src.shape, dtype=kind.torch_dtype, device=src.device)
    flag = torch.zeros(1, dtype=torch.int32, device=src.device) if check else None
    if src.numel():
        _native.call("bz_round_to_kind", src.data_ptr(), kind_of_dtype(src.dtype).code,
                     out.data_ptr(), kind.code, src.numel(),
                     flag.data_ptr() if check else None, _stream(src))
    if check and int(flag.item()):
        raise ValueError(f"values are not exactly representable as {kind.value}")
    return out


class DenseArray:
    """An N-dimensional array of `kind` values held on the GPU.

    Constructing from a buffer copies it (the reference freezes its own copy,
    arrays.py:51-62); values must already be representable in `kind`
    (ValueError otherwise, arrays.py:81-86).  Use :meth:`of` to round.
    """

    __slots__ = ("shape", "kind", "values")

    def __init__(self, shape, kind: FloatKind, values, *, _trusted: bool = False):
        shape = validate_shape(shape)
        if _trusted:
            t = values
        else:
            src = as_device_tensor(values)
            if tuple(src.shape) != shape:
                raise DimensionMismatch(
                    f"value buffer shaped {tuple(src.shape)} does not match shape {shape}"
                )
            # a copy in the kind's dtype; narrowing is checked to be exact
            if src.dtype == kind.torch_dtype:
                fresh = not (isinstance(values, torch.Tensor) and values.is_cuda
                             and values.data_ptr() == src.data_ptr())
                t = src if fresh else src.clone()  # host data was already copied once
            else:
                t = _round_into(src, kind, check=True)
        object.__setattr__(self, "shape", shape)
        object.__setattr__(self, "kind", kind)
        object.__setattr__(self, "values", t)

    def __setattr__(self, name, value):
        raise AttributeError("DenseArray is immutable")

    @classmethod
    def of(cls, values, kind: FloatKind = FloatKind.F64) -> "DenseArray":
        """Round arbitrary values into `kind` (arrays.py:89-93)."""
        src = as_device_tensor(values)
        shape = validate_shape(src.shape) if src.dim() else validate_shape((1,))
        return cls(shape, kind, _round_into(src.reshape(shape), kind, check=False), _trusted=True)

    @classmethod
    def wrap(cls, tensor: torch.Tensor, kind: FloatKind | None = None) -> "DenseArray":
        """Adopt a contiguous CUDA tensor of a float kind's dtype without copying.

        The caller promises not to mutate it afterwards (zero-copy entry for
        large resident inputs).
        """
        k = kind_of_dtype(tensor.dtype) if kind is None else kind
        if k is None or tensor.dtype != k.torch_dtype or not tensor.is_cuda:
            raise ValueError("wrap() needs a CUDA tensor in the kind's native dtype")
        return cls(tuple(tensor.shape), k, tensor.contiguous(), _trusted=True)

    @property
    def ndim(self) -> int:
        return len(self.shape)

    @property
    def size(self) -> int:
        return int(np.prod(self.shape))

    def numpy(self) -> np.ndarray:
        """float64 host copy (the reference's value representation)."""
        return self.values.to(torch.float64).cpu().numpy()

    def __repr__(self):
        return f"DenseArray(shape={self.shape}, kind={self.kind.value}, device={self.values.device})"


class BlockedArray:
    """A dense array cut into zero-padded blocks: float64 ``grid + block`` tensor."""

    __slots__ = ("block_grid", "block_shape", "original_shape", "kind", "blocks")

    def __init__(self, block_grid, block_shape, original_shape, kind: FloatKind, blocks,
                 *, _trusted: bool = False):
        grid = validate_shape(block_grid)
        bshape = validate_shape(block_shape)
        orig = validate_shape(original_shape)
        if not (len(grid) == len(bshape) == len(orig)):
            raise DimensionMismatch("grid, block and original shapes disagree on rank")
        if grid != grid_shape(orig, bshape):
            raise DimensionMismatch(f"grid {grid} is not ceil({orig} / {bshape})")
        if _trusted:
            t = blocks
        else:
            t = as_device_tensor(blocks).to(torch.float64).clone()
        if tuple(t.shape) != grid + bshape:
            raise DimensionMismatch(f"block buffer shaped {tuple(t.shape)}, expected {grid + bshape}")
        for name, v in (("block_grid", grid), ("block_shape", bshape), ("original_shape", orig),
                        ("kind", kind), ("blocks", t)):
            object.__setattr__(self, name, v)

    def __setattr__(self, name, value):
        raise AttributeError("BlockedArray is immutable")

    @property
    def ndim(self) -> int:
        return len(self.block_shape)

    @property
    def block_count(self) -> int:
        return int(np.prod(self.block_grid))


def _plain_layout(shape, block_shape) -> _native.Layout:
    """Layout without codec tables (blocking only)."""
    L = _native.Layout()
    L.ndim = len(shape)
    L.float_kind = FloatKind.F64.code
    L.index_kind = 0
    L.transform = 0
    for a, (s, b) in enumerate(zip(shape, block_shape)):
        L.shape[a] = s
        L.block[a] = b
        L.grid[a] = -(-s // b)
    L.kept = 0
    L.keeps_first = 0
    return L


def convert_precision(a: DenseArray, kind: FloatKind) -> DenseArray:
    """Round every element into `kind` (arrays.py:147-153)."""
    return DenseArray(a.shape, kind, _round_into(a.values, kind, check=False), _trusted=True)


def _check_block(a_ndim: int, block_shape) -> tuple[int, ...]:
    bshape = validate_shape(block_shape)
    if len(bshape) != a_ndim:
        raise DimensionMismatch(
            f"block shape {bshape} has rank {len(bshape)}, array has rank {a_ndim}"
        )
    if not all(is_power_of_two(b) for b in bshape):
        raise NonPowerOfTwoBlock(f"block extents must be powers of two, got {bshape}")
    return bshape


def block(a: DenseArray, block_shape) -> BlockedArray:
    """Zero-pad and regroup into ``grid + block`` (arrays.py:156-178), on the GPU."""
    bshape = _check_block(a.ndim, block_shape)
    grid = grid_shape(a.shape, bshape)
    out = torch.empty(grid + bshape, dtype=torch.float64, device=a.values.device)
    L = _plain_layout(a.shape, bshape)
    _native.call("bz_block", _native.ctypes.byref(L), a.values.data_ptr(), a.kind.code,
                 out.data_ptr(), _stream(out))
    return BlockedArray(grid, bshape, a.shape, a.kind, out, _trusted=True)


def unblock(b: BlockedArray) -> DenseArray:
    """Merge blocks and crop (arrays.py:181-190); exact inverse of block."""
    out = torch.empty(b.original_shape, dtype=b.kind.torch_dtype, device=b.blocks.device)
    L = _plain_layout(b.original_shape, b.block_shape)
    _native.call("bz_unblock", _native.ctypes.byref(L), b.blocks.data_ptr(), out.data_ptr(),
                 b.kind.code, _stream(out))
    return DenseArray(b.original_shape, b.kind, out, _trusted=True)


def gradient_array(shape, kind: FloatKind = FloatKind.F64) -> DenseArray:
    """Element x = sum(x) / sum(shape-1), zero-based (arrays.py:193-208)."""
    dims = validate_shape(shape)
    if sum(d - 1 for d in dims) == 0:
        raise DegenerateShape(f"gradient over {dims} needs an extent > 1")
    out = torch.empty(dims, dtype=kind.torch_dtype, device=torch.device("cuda", torch.cuda.current_device()))
    arr = (_native.ctypes.c_int64 * len(dims))(*dims)
    _native.call("bz_gradient", len(dims), arr, kind.code, out.data_ptr(), _stream(out))
    return DenseArray(dims, kind, out, _trusted=True)
