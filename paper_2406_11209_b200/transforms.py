"""Orthonormal block transforms (reference: pkg/src/bzc/transforms.py).

Matrix entries are built on the host with the reference's own float64
expressions (transforms.py:67-81), so they are bit-identical; they are
uploaded once per settings and used by the generic kernels.  The fused
compress/decompress kernels use factored butterflies of the same bases
(csrc/bz_transforms.cuh).
"""

from __future__ import annotations

import enum
import functools
import math

import numpy as np
import torch

from . import _native
from .arrays import BlockedArray, is_power_of_two
from .errors import DimensionMismatch, NonPowerOfTwoBlock

__all__ = [
    "TransformFamily",
    "TransformMatrix",
    "make_transform",
    "transforms_for",
    "forward_transform",
    "inverse_transform",
]


class TransformFamily(enum.Enum):
    DCT = "dct"
    HAAR = "haar"

    @property
    def code(self) -> int:
        return 0 if self is TransformFamily.DCT else 1

    @classmethod
    def from_code(cls, code: int) -> "TransformFamily":
        return cls.DCT if code == 0 else cls.HAAR

    @classmethod
    def parse(cls, name: str) -> "TransformFamily":
        return cls(name.strip().lower())


class TransformMatrix:
    """One per-axis orthonormal basis, entries [sample, basis] (host float64)."""

    __slots__ = ("size", "family", "entries")

    def __init__(self, size: int, family: TransformFamily, entries):
        e = np.array(entries, dtype=np.float64, copy=True)
        e.flags.writeable = False
        object.__setattr__(self, "size", int(size))
        object.__setattr__(self, "family", family)
        object.__setattr__(self, "entries", e)

    def __setattr__(self, name, value):
        raise AttributeError("TransformMatrix is immutable")

    def __eq__(self, other):
        return (isinstance(other, TransformMatrix) and self.size == other.size
                and self.family is other.family and np.array_equal(self.entries, other.entries))

    def __hash__(self):
        return hash((self.size, self.family))


def _dct_entries(size: int) -> np.ndarray:
    # same float64 expression as the reference (and the paper's H formula)
    samples = np.arange(size, dtype=np.float64)[:, None]
    basis = np.arange(size, dtype=np.float64)[None, :]
    scale = np.sqrt((1.0 + (basis > 0)) / size)
    return scale * np.cos(np.pi * basis * (2.0 * samples + 1.0) / (2.0 * size))


def _haar_entries(size: int) -> np.ndarray:
    # coarse-to-fine Haar: level-by-level halvings, entries +-(1/sqrt2)^t by
    # repeated IEEE division (bit-identical to the reference construction,
    # including -0.0 in the lower half of each wavelet's zero rows)
    levels = int(round(math.log2(size)))
    mag = [1.0]
    for _ in range(levels):
        mag.append(mag[-1] / np.sqrt(2.0))
    h = np.zeros((size, size))
    h[:, 0] = mag[levels]
    col = 1
    for lvl in range(levels):
        count = 1 << lvl
        half = size // count // 2
        for j in range(count):
            for row in range(size):
                coarse = row // half
                v = mag[levels - lvl] if (coarse >> 1) == j else 0.0
                h[row, col] = -v if (coarse & 1) else v
            col += 1
    return h


@functools.lru_cache(maxsize=None)
def _entries(size: int, family: TransformFamily) -> np.ndarray:
    e = _dct_entries(size) if family is TransformFamily.DCT else _haar_entries(size)
    e.flags.writeable = False
    return e


def make_transform(size: int, family: TransformFamily) -> TransformMatrix:
    """Orthonormal basis of `family` for one block extent (transforms.py:94-98)."""
    if not is_power_of_two(size):
        raise NonPowerOfTwoBlock(f"transform size must be a power of two, got {size}")
    return TransformMatrix(size, family, _entries(size, family))


def transforms_for(block_shape, family: TransformFamily) -> tuple[TransformMatrix, ...]:
    return tuple(make_transform(s, family) for s in block_shape)


def _check_mats(block_shape, mats) -> None:
    if len(mats) != len(block_shape):
        raise DimensionMismatch(f"{len(mats)} matrices for {len(block_shape)} block axes")
    sizes = tuple(m.size for m in mats)
    if sizes != tuple(block_shape):
        raise DimensionMismatch(f"matrix sizes {sizes} do not match block shape {tuple(block_shape)}")


def matrices_tensor(mats, device) -> torch.Tensor:
    flat = np.concatenate([m.entries.reshape(-1) for m in mats])
    return torch.from_numpy(flat).to(device)


def _run(b: BlockedArray, mats, inverse: int) -> BlockedArray:
    _check_mats(b.block_shape, mats)
    dev = b.blocks.device
    mt = matrices_tensor(mats, dev)
    L = _native.Layout()
    L.ndim = len(b.block_shape)
    L.float_kind = 3
    for a, (s, i) in enumerate(zip(b.original_shape, b.block_shape)):
        L.shape[a] = s
        L.block[a] = i
        L.grid[a] = -(-s // i)
    L.matrices = mt.data_ptr()
    out = torch.empty_like(b.blocks)
    ws = torch.empty(b.blocks.numel() * 8 if L.ndim > 1 else 8, dtype=torch.uint8, device=dev)
    _native.call("bz_transform", _native.ctypes.byref(L), b.blocks.contiguous().data_ptr(),
                 out.data_ptr(), inverse, ws.data_ptr(), ws.numel(), _native.stream_handle(dev))
    return BlockedArray(b.block_grid, b.block_shape, b.original_shape, b.kind, out, _trusted=True)


def forward_transform(b: BlockedArray, mats) -> BlockedArray:
    """Coefficients of every block in the per-axis bases (transforms.py:129-134)."""
    return _run(b, mats, 0)


def inverse_transform(c: BlockedArray, mats) -> BlockedArray:
    """Blocks rebuilt from coefficients (transforms.py:137-142)."""
    return _run(c, mats, 1)
