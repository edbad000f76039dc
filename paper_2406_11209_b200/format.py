"""Bit-exact ``.bzc`` streams of compressed arrays (reference: format.py).

Same API as the reference module -- ``BitstreamLayout``, ``bitstream_layout``,
``serialize``, ``deserialize`` -- and the same stream, bit for bit
(format.py:1-33): LSB-first bits, little-endian fields; float kind (2 bits),
index kind (2), transform (8), original shape (64 per extent), a zero word,
block shape (64 per extent), the pruning mask (1 bit per position), maxima
(raw patterns), indices (two's complement), zero padding to a byte.

The header is a few hundred bits and is built on the host.  The payload --
maxima then indices, which is exactly their little-endian bytes shifted to
the header's bit offset -- is packed and unpacked on the GPU by
``bz_stream_pack`` / ``bz_stream_unpack`` (csrc/bz_format.cu).
``serialize_to_device`` returns the stream as a CUDA uint8 tensor without a
host round trip; ``serialize`` copies it to ``bytes``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .codec import CodecSettings, CompressedArray, PruningMask, _device
from .errors import InvalidTypeCode, TruncatedStream, ZeroExtent
from .kinds import FloatKind, IndexKind
from .transforms import TransformFamily

__all__ = ["BitstreamLayout", "bitstream_layout", "serialize", "serialize_to_device",
           "deserialize"]

_SHAPE_WORD_BITS = 64


@dataclass(frozen=True)
class BitstreamLayout:
    """Ordered (field name, bit offset, bit length) records for one stream."""

    fields: tuple[tuple[str, int, int], ...]

    @property
    def content_bits(self) -> int:
        name, offset, _ = self.fields[-1]
        assert name == "padding"
        return offset

    @property
    def total_bits(self) -> int:
        _, offset, length = self.fields[-1]
        return offset + length

    @property
    def total_bytes(self) -> int:
        return self.total_bits // 8


def _fields(settings: CodecSettings, ndim: int, blocks: int):
    fields, pos = [], 0
    for name, length in (
        ("float_kind", 2),
        ("index_kind", 2),
        ("transform", 8),
        ("original_shape", _SHAPE_WORD_BITS * ndim),
        ("shape_marker", _SHAPE_WORD_BITS),
        ("block_shape", _SHAPE_WORD_BITS * ndim),
        ("mask", settings.block_size),
        ("maxima", settings.float_kind.bits * blocks),
        ("indices", settings.index_kind.bits * settings.mask.kept_count * blocks),
    ):
        fields.append((name, pos, length))
        pos += length
    fields.append(("padding", pos, (-pos) % 8))
    return tuple(fields)


def bitstream_layout(a: CompressedArray) -> BitstreamLayout:
    """Field offsets of ``a``'s stream (format.py:91-92)."""
    return BitstreamLayout(_fields(a.settings, a.settings.ndim, a.block_count))


def _header_bits(a: CompressedArray) -> np.ndarray:
    """The header as an LSB-first bit array (host; a few hundred bits)."""
    s = a.settings

    def bits_of(values, width):
        vals = np.asarray(values, dtype=np.uint64).ravel()
        shifts = np.arange(width, dtype=np.uint64)
        return ((vals[:, None] >> shifts[None, :]) & np.uint64(1)).astype(np.uint8).ravel()

    mask_bits = np.asarray(s.mask.bits)
    return np.concatenate([
        bits_of([s.float_kind.code], 2),
        bits_of([s.index_kind.code], 2),
        bits_of([s.transform.code], 8),
        bits_of(list(a.original_shape), _SHAPE_WORD_BITS),
        bits_of([0], _SHAPE_WORD_BITS),
        bits_of(list(s.block_shape), _SHAPE_WORD_BITS),
        mask_bits.ravel().astype(np.uint8),
    ])


def serialize_to_device(a: CompressedArray) -> torch.Tensor:
    """The stream as a CUDA uint8 tensor (payload packed on the GPU)."""
    layout = bitstream_layout(a)
    head = _header_bits(a)
    P = head.size
    total = layout.total_bytes
    nwords = (total + 3) // 4
    dev = a.device
    out = torch.empty(nwords * 4, dtype=torch.uint8, device=dev)
    # whole header words on the host; the partial word goes to the kernel
    full = P // 32
    hw = np.zeros((full + 1) * 32, dtype=np.uint8)
    hw[:P] = head
    words = np.packbits(hw, bitorder="little").view("<u4")
    if full:
        out[: full * 4].copy_(torch.from_numpy(words[:full].view(np.uint8).copy()), non_blocking=True)
    maxima = a.maxima.contiguous()
    indices = a.indices.contiguous()
    _native.call("bz_stream_pack", maxima.data_ptr(), maxima.numel() * maxima.element_size(),
                 indices.data_ptr(), indices.numel() * indices.element_size(), P,
                 int(words[full]), out.data_ptr(), nwords, _native.stream_handle(dev))
    return out[:total]


def serialize(a: CompressedArray) -> bytes:
    """Encode a compressed array as its byte stream (format.py:108-127)."""
    return serialize_to_device(a).cpu().numpy().tobytes()


class _Reader:
    """Header reader over the first bytes of a stream (format.py:130-162)."""

    def __init__(self, head: np.ndarray, total_bits: int):
        self.bits = np.unpackbits(head, bitorder="little")
        self.total = total_bits
        self.pos = 0

    def take(self, n: int) -> np.ndarray:
        if self.pos + n > self.total:
            raise TruncatedStream(f"needed {n} bits at offset {self.pos}, stream has {self.total}")
        if self.pos + n > self.bits.size:
            raise TruncatedStream(f"header longer than {self.bits.size} bits")
        out = self.bits[self.pos:self.pos + n]
        self.pos += n
        return out

    def uint(self, width: int) -> int:
        bits = self.take(width)
        return int(sum(int(b) << j for j, b in enumerate(bits)))


def parse_header(head: np.ndarray, total_bytes: int):
    """Parse a stream's header on the host (format.py:165-188): returns
    (shape, CodecSettings, payload bit offset).  Raises TruncatedStream,
    InvalidTypeCode or ZeroExtent exactly as the reference."""
    r = _Reader(np.asarray(head, dtype=np.uint8), total_bytes * 8)
    float_kind = FloatKind.from_code(r.uint(2))
    index_kind = IndexKind.from_code(r.uint(2))
    transform_code = r.uint(8)
    if transform_code not in (0, 1):
        raise InvalidTypeCode(f"unknown transform code {transform_code}")
    transform = TransformFamily.from_code(transform_code)
    shape = []
    while True:
        word = r.uint(_SHAPE_WORD_BITS)
        if word == 0:
            break
        shape.append(word)
    if not shape:
        raise ZeroExtent("shape is empty (zero extent before any valid extent)")
    d = len(shape)
    block_shape = [r.uint(_SHAPE_WORD_BITS) for _ in range(d)]
    if any(b == 0 for b in block_shape):
        raise ZeroExtent(f"block shape {tuple(block_shape)} contains a zero extent")
    mask_bits = r.take(math.prod(block_shape))
    mask = PruningMask.from_bits(tuple(block_shape), mask_bits.astype(bool))
    settings = CodecSettings(tuple(block_shape), float_kind, index_kind, transform, mask)
    P = r.pos
    grid = settings.grid_for(tuple(shape))
    blocks = math.prod(grid)
    payload_bits = 8 * blocks * (float_kind.itemsize + mask.kept_count * index_kind.itemsize)
    if P + payload_bits > total_bytes * 8:
        raise TruncatedStream(f"needed {payload_bits} payload bits at offset {P}, "
                              f"stream has {total_bytes * 8}")
    return tuple(shape), settings, P


def deserialize(data) -> CompressedArray:
    """Decode a stream (bytes, bytearray, numpy uint8 or a uint8 tensor).

    The header is parsed on the host; the payload is unpacked on the GPU.
    Raises TruncatedStream, InvalidTypeCode or ZeroExtent on malformed input
    (format.py:165-209), before any device work.
    """
    if isinstance(data, torch.Tensor):
        stream = data.reshape(-1)
        if stream.dtype != torch.uint8:
            raise TypeError("stream tensor must be uint8")
        host_head = stream[:1 << 20].cpu().numpy()
        nbytes = stream.numel()
    else:
        buf = np.frombuffer(bytes(data), dtype=np.uint8)
        stream = None
        host_head = buf[:1 << 20]
        nbytes = buf.size
    shape, settings, P = parse_header(host_head, nbytes)
    grid = settings.grid_for(shape)
    blocks = math.prod(grid)
    kept = settings.mask.kept_count
    max_bytes = blocks * settings.float_kind.itemsize
    idx_bytes = blocks * kept * settings.index_kind.itemsize
    dev = stream.device if (stream is not None and stream.is_cuda) else _device()
    nwords = (nbytes + 3) // 4
    words = torch.zeros(nwords * 4, dtype=torch.uint8, device=dev)
    if stream is not None:
        words[:nbytes].copy_(stream)
    else:
        words[:nbytes].copy_(torch.from_numpy(buf.copy()))
    maxima = torch.empty(grid, dtype=settings.float_kind.torch_dtype, device=dev)
    indices = torch.empty(tuple(grid) + (kept,), dtype=settings.index_kind.torch_dtype, device=dev)
    _native.call("bz_stream_unpack", words.data_ptr(), nwords, P, maxima.data_ptr(), max_bytes,
                 indices.data_ptr(), idx_bytes, _native.stream_handle(dev))
    return CompressedArray(shape, settings, maxima, indices)
