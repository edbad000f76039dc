"""Multi-process (world_size 2, gloo, CPU) tests of the block-sharded path.

The partition, the record exchange (all_gather over the process group) and
the Chan merge + epilogue run exactly as on the GPUs; only the per-shard
record comes from a numpy restatement of the bz_moments definition (no GPU
here).  Results must match the oracle on the unsharded array.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bzc_oracle as o

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def np_record(a_max, a_idx, b_max, b_idx, keeps_first, dc_only):
    """Numpy restatement of one shard's bz_moments record (include/bzc_b200.h)."""
    k = a_idx.shape[-1]
    fa = a_idx.reshape(-1, k).astype(np.float64)
    fb = b_idx.reshape(-1, k).astype(np.float64)
    na, nb = a_max.reshape(-1), b_max.reshape(-1)
    n = fa.shape[0]
    rec = np.zeros(16)
    rec[0] = n
    if dc_only == 2:  # "sums" (dot / l2): every kept position goes into S_*
        keeps_first, dc_only = False, 0
    if keeps_first and k:
        dca, dcb = fa[:, 0] * na, fb[:, 0] * nb
        ma, mb = dca.mean(), dcb.mean()
        rec[1:6] = [ma, mb, np.sum((dca - ma) * (dcb - mb)), np.sum((dca - ma) ** 2),
                    np.sum((dcb - mb) ** 2)]
        fa, fb = fa[:, 1:], fb[:, 1:]
    if not dc_only:
        rec[6] = np.sum(na * nb * np.sum(fa * fb, axis=1))
        rec[7] = np.sum(na * na * np.sum(fa * fa, axis=1))
        rec[8] = np.sum(nb * nb * np.sum(fb * fb, axis=1))
    return torch.from_numpy(rec)


def _worker(rank, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_2406_11209_b200 as bz
        from paper_2406_11209_b200 import distributed as bd

        shape, block = (37, 24, 16), (8, 8, 8)
        rng = np.random.default_rng(123)
        xa = rng.uniform(0, 1, shape)
        xb = 0.5 * xa + 0.5 * rng.uniform(0, 1, shape)
        os_ = o.Settings(block, "f32", "i8")
        ra = o.compress(o.round_to_kind(xa, "f32"), os_)
        rb = o.compress(o.round_to_kind(xb, "f32"), os_)

        r0, r1 = bd.shard_slab(shape, block, rank, WORLD)
        b0, b1 = bd.block_rows(ra.maxima.shape[0], rank, WORLD)
        assert b0 * 8 == r0 and (b1 * 8 >= r1)
        s = bz.CodecSettings(block, bz.FloatKind.F32, bz.IndexKind.I8)
        local_shape = (r1 - r0,) + shape[1:]

        def shard(r):
            m = torch.from_numpy(r.maxima[b0:b1].astype(np.float32))
            i = torch.from_numpy(r.indices[b0:b1])
            return bz.CompressedArray(local_shape, s, m, i, _trusted=True)

        def rec_fn(a, b, dc_only):
            bb = a if b is None else b
            return np_record(a.maxima.double().numpy(), a.indices.numpy(),
                             bb.maxima.double().numpy(), bb.indices.numpy(),
                             a.settings.mask.keeps_first, dc_only)

        a = bd.ShardedCompressedArray(shard(ra), shape, record_fn=rec_fn)
        b = bd.ShardedCompressedArray(shard(rb), shape, record_fn=rec_fn)
        got = {
            "dot": bz.dot(a, b), "l2": bz.l2_norm(a), "mean": bz.mean(a),
            "mean_pc": bz.mean(a, padding_corrected=True), "var": bz.variance(a),
            "cov": bz.covariance(a, b), "cos": bz.cosine_similarity(a, b), "ssim": bz.ssim(a, b),
        }
        want = {
            "dot": o.dot(ra, rb), "l2": o.l2_norm(ra), "mean": o.mean(ra),
            "mean_pc": o.mean(ra, True), "var": o.variance(ra), "cov": o.covariance(ra, rb),
            "cos": o.cosine_similarity(ra, rb), "ssim": o.ssim(ra, rb),
        }
        results[rank] = (got, want)
    finally:
        dist.destroy_process_group()


def test_sharded_reductions_match_unsharded_oracle():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, results)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert set(results.keys()) == set(range(WORLD))
    g0, _ = results[0]
    for r in range(WORLD):
        got, want = results[r]
        assert got == g0  # every rank returns the same value
        for k in want:
            assert math.isclose(got[k], want[k], rel_tol=1e-9, abs_tol=1e-12), (k, got[k], want[k])


def test_partition_covers_the_array():
    from paper_2406_11209_b200 import distributed as bd

    for shape, block, world in (((1024, 8), (8, 8), 8), ((37, 5), (8, 4), 4), ((5, 3), (4, 1), 8)):
        rows = [bd.shard_slab(shape, block, r, world) for r in range(world)]
        assert rows[0][0] == 0 and rows[-1][1] == shape[0]
        for (a0, a1), (c0, c1) in zip(rows, rows[1:]):
            assert a1 == c0 and a0 <= a1
            assert a1 % block[0] == 0 or a1 == shape[0]
