"""Block-sharded arrays over the GPUs of one node.

One process per GPU (``torch.distributed``, NCCL over NVLink/NVSwitch).  The
block grid is split along grid axis 0 into contiguous block-row ranges
``[floor(G0*g/P), floor(G0*(g+1)/P))``; shard g owns the dense slab
``[i0*start, min(i0*end, s0))`` of axis 0.  Compress, decompress and every
elementwise operator are shard-local (blocks are independent,
PAPER.md:295) -- no communication.  A reduction computes the shard's partial
record with the fused ``bz_moments`` kernel, all-gathers the P records
(P x 16 float64 -- the only data that crosses NVLink) and merges them in rank
order with Chan's formulas, so every rank returns the same value (one
all_gather_into_tensor and one device->host copy per reduction).  The
concatenation of the shards' maxima / indices along axis 0 is exactly the
unsharded CompressedArray.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .arrays import DenseArray, grid_shape, validate_shape
from .codec import CodecSettings, CompressedArray, compress as _compress
from .ops import Record, merge_records, moments_record

__all__ = ["block_rows", "shard_slab", "ShardedCompressedArray", "compress_sharded",
           "gather_records", "allgather_sum"]


def block_rows(g0: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block-row range of `rank` out of `world` over g0 block rows."""
    return (g0 * rank) // world, (g0 * (rank + 1)) // world


def shard_slab(global_shape, block_shape, rank: int, world: int) -> tuple[int, int]:
    """Dense row range [r0, r1) along axis 0 owned by `rank`."""
    g0 = grid_shape(global_shape, block_shape)[0]
    b0, b1 = block_rows(g0, rank, world)
    i0 = int(block_shape[0])
    return b0 * i0, min(b1 * i0, int(global_shape[0]))


def gather_records(rec: torch.Tensor, group=None) -> list[Record]:
    """One collective per reduction: all-gather every rank's 16-double record
    into one (P*16) tensor (NCCL over NVLink on GPU tensors, gloo on CPU),
    then ONE device->host copy; the P records are merged on the host in rank
    order (P <= 8 records -- microseconds)."""
    world = dist.get_world_size(group)
    flat = rec.contiguous().reshape(-1)
    if dist.get_backend(group) != "nccl" and flat.is_cuda:
        flat = flat.cpu()  # gloo moves host tensors
    out = torch.empty(world * flat.numel(), dtype=flat.dtype, device=flat.device)
    dist.all_gather_into_tensor(out, flat, group=group)
    host = out.cpu().numpy().reshape(world, -1)
    return [Record.from_array(host[r]) for r in range(world)]


def allgather_sum(x: torch.Tensor, group=None) -> float:
    """Sum of one double per rank, added in rank order (deterministic)."""
    world = dist.get_world_size(group)
    x = x.reshape(1).to(torch.float64)
    if dist.get_backend(group) != "nccl" and x.is_cuda:
        x = x.cpu()
    out = torch.empty(world, dtype=torch.float64, device=x.device)
    dist.all_gather_into_tensor(out, x, group=group)
    return float(sum(float(v) for v in out.cpu().numpy()))


class ShardedCompressedArray(CompressedArray):
    """This rank's shard of a block-sharded compressed array.

    ``original_shape`` is the local slab's shape (what the kernels see);
    ``global_shape`` is the whole array's.  The operators in ``ops`` accept
    it unchanged: reductions merge records across the group first, and
    elementwise results stay sharded.
    """

    __slots__ = ("global_shape", "group", "_record_fn")

    def __init__(self, local: CompressedArray, global_shape, group=None, record_fn=None):
        super().__init__(local.original_shape, local.settings, local.maxima, local.indices,
                         _trusted=True, dc=local.dc_plane)
        object.__setattr__(self, "global_shape", validate_shape(global_shape))
        object.__setattr__(self, "group", group)
        object.__setattr__(self, "_record_fn", record_fn or _device_record)

    def _derive(self, maxima, indices, dc=None):
        local = CompressedArray(self.original_shape, self.settings, maxima, indices, _trusted=True,
                                dc=dc)
        return ShardedCompressedArray(local, self.global_shape, self.group, self._record_fn)

    def _reduce_record(self, b, dc_only):
        other = None if b is None or b is self else b
        rec = self._record_fn(self, other, dc_only)
        return merge_records(gather_records(rec, self.group))

    def _reduce_sum(self, x: torch.Tensor) -> float:
        return allgather_sum(x, self.group)

    @property
    def local(self) -> CompressedArray:
        return CompressedArray(self.original_shape, self.settings, self.maxima, self.indices,
                               _trusted=True, dc=self.dc_plane)


def _device_record(a, b, dc_only):
    plain_a = CompressedArray(a.original_shape, a.settings, a.maxima, a.indices, _trusted=True,
                              dc=a.dc_plane)
    plain_b = None if b is None else CompressedArray(b.original_shape, b.settings, b.maxima,
                                                     b.indices, _trusted=True, dc=b.dc_plane)
    return moments_record(plain_a, plain_b, dc_only=dc_only)


def compress_sharded(local: DenseArray, settings: CodecSettings, global_shape,
                     group=None) -> ShardedCompressedArray:
    """Compress this rank's slab; the slab must be block-row aligned (shard_slab)."""
    global_shape = validate_shape(global_shape)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    r0, r1 = shard_slab(global_shape, settings.block_shape, rank, world)
    if tuple(local.shape) != (r1 - r0,) + tuple(global_shape[1:]):
        raise ValueError(f"rank {rank} slab shape {local.shape} != expected "
                         f"{(r1 - r0,) + tuple(global_shape[1:])}")
    return ShardedCompressedArray(_compress(local, settings), global_shape, group)


def concat_shards(shards: list[CompressedArray], global_shape) -> CompressedArray:
    """Reassemble the unsharded CompressedArray (testing / gathering)."""
    s = shards[0].settings
    m = torch.cat([x.maxima.to(shards[0].device) for x in shards], dim=0)
    i = torch.cat([x.indices.to(shards[0].device) for x in shards], dim=0)
    dc = None
    if all(x.dc_plane is not None for x in shards):
        dc = torch.cat([x.dc_plane.to(shards[0].device) for x in shards], dim=0)
    return CompressedArray(tuple(global_shape), s, m, i, _trusted=True, dc=dc)


def expected_partition(global_shape, block_shape, world: int) -> list[tuple[int, int]]:
    return [shard_slab(global_shape, block_shape, r, world) for r in range(world)]


def np_slab(values: np.ndarray, block_shape, rank: int, world: int) -> np.ndarray:
    r0, r1 = shard_slab(values.shape, block_shape, rank, world)
    return values[r0:r1]
