"""Per-kernel timings for the BASELINE configs (CUDA events, inputs > L2).

Usage: python tools/quick_bench.py [c1 c2 c3 c4 c5 ...]
Prints one line per op: ms, GB/s of uncompressed input, algorithmic GB/s and
the fraction of the measured HBM peak.
"""

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2406_11209_b200 as bz  # noqa: E402
from paper_2406_11209_b200 import _native  # noqa: E402


def peak_gbs():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        return 6650.0


def fill(shape, kind, seed, dist=0):
    t = torch.empty(shape, dtype=kind.torch_dtype, device="cuda")
    _native.call("bz_fill_random", t.data_ptr(), kind.code, t.numel(), 0, seed, dist,
                 _native.stream_handle())
    return bz.DenseArray.wrap(t, kind)


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


CONFIGS = {
    "c1": ((256, 256, 256), (8, 8, 8), "f32", "i8", None),
    "c2": ((8192, 8192), (4, 4), "f64", "i16", None),
    "c3": ((1024, 1024, 1024), (8, 8, 8), "f32", "i8", None),
    "c5": ((256, 256, 256, 64), (4, 4, 4, 4), "f32", "i8", "lowpass"),
    "c4": ((1024, 1024, 1024), (8, 8, 8), "f32", "i8", None),  # uniform data (dist 1)
    "c2x4": ((16384, 16384), (4, 4), "f64", "i16", None),      # tail-cost probe
}


def run(name):
    shape, block, fk, ik, mask = CONFIGS[name]
    bits = (np.indices(block).sum(axis=0) <= 4) if mask == "lowpass" else None
    s = bz.CodecSettings(block, bz.FloatKind(fk), bz.IndexKind(ik),
                         mask=None if bits is None else bz.PruningMask(block, bits))
    kind = bz.FloatKind(fk)
    dist = 1 if name == "c4" else 0
    x = fill(shape, kind, 1, dist)
    y = fill(shape, kind, 2, dist)
    n = x.values.numel()
    inb = n * kind.itemsize
    B = int(np.prod(s.grid_for(shape)))
    K = s.mask.kept_count
    comp_bytes = B * (K * s.index_kind.itemsize + kind.itemsize)
    peak = peak_gbs()
    ca = bz.compress(x, s)
    cb = bz.compress(y, s)
    rows = []

    only = [o for o in os.environ.get("QB_OPS", "").split(",") if o]

    def timeit_(fn, reps=10, warm=3):
        return timeit(fn, reps, warm)

    def rec_(op, ms_thunk_or_ms, alg_bytes, in_bytes=inb):
        if only and op not in only:
            return
        rec(op, ms_thunk_or_ms() if callable(ms_thunk_or_ms) else ms_thunk_or_ms, alg_bytes,
            in_bytes)

    def rec(op, ms, alg_bytes, in_bytes=inb):
        rows.append((op, ms, in_bytes / ms / 1e6, alg_bytes / ms / 1e6, alg_bytes / ms / 1e6 / peak))

    rec_("compress", lambda: timeit(lambda: bz.compress(x, s)), inb + comp_bytes)
    rec_("decompress_f64", lambda: timeit(lambda: bz.decompress(ca)), comp_bytes + n * 8)
    rec_("decompress_fk", lambda: timeit(lambda: bz.decompress(ca, kind)), comp_bytes + n * kind.itemsize)
    rec_("l2_record", lambda: timeit(lambda: bz.ops.moments_record(ca, dc_only=2)), comp_bytes)
    rec_("dot_record", lambda: timeit(lambda: bz.ops.moments_record(ca, cb, dc_only=2)), 2 * comp_bytes, 2 * inb)
    if s.mask.keeps_first:
        rec_("cov_record", lambda: timeit(lambda: bz.ops.moments_record(ca, cb)), 2 * comp_bytes, 2 * inb)
        rec_("mean_record", lambda: timeit(lambda: bz.ops.moments_record(ca, dc_only=1)),
             B * (s.index_kind.itemsize + kind.itemsize))
    rec_("add", lambda: timeit(lambda: bz.add(ca, cb)), 3 * comp_bytes, 2 * inb)
    rec_("negate", lambda: timeit(lambda: bz.negate(ca)), 2 * B * K * s.index_kind.itemsize)
    rec_("l2_norm(api)", lambda: timeit(lambda: bz.l2_norm(ca)), comp_bytes)
    rec_("mean(api)", lambda: timeit(lambda: bz.mean(ca)), B * (s.index_kind.itemsize + kind.itemsize))
    if s.mask.keeps_first:
        rec_("cov(api)", lambda: timeit(lambda: bz.covariance(ca, cb)), 2 * comp_bytes, 2 * inb)
        rec_("ssim(api)", lambda: timeit(lambda: bz.ssim(ca, cb)), 2 * comp_bytes, 2 * inb)
        rec_("subtract_l2", lambda: timeit(lambda: bz.subtract_l2(cb, ca)), 2 * comp_bytes, 2 * inb)
        rec_("wasserstein", lambda: timeit(lambda: bz.approx_wasserstein(ca, cb), reps=3, warm=1),
            2 * B * (s.index_kind.itemsize + kind.itemsize))
    rec_("serialize_dev", lambda: timeit(lambda: bz.serialize_to_device(ca)), 2 * comp_bytes)
    print(f"== {name} shape={shape} block={block} {fk}/{ik} K={K} fast={bz.is_fast_path(s, shape)}")
    for op, ms, g_in, g_alg, frac in rows:
        print(f"  {op:16s} {ms*1e3:9.1f} us  in {g_in:8.0f} GB/s  alg {g_alg:7.0f} GB/s  frac {frac:.3f}")
    sys.stdout.flush()


if __name__ == "__main__":
    for name in (sys.argv[1:] or ["c2", "c1", "c3", "c5"]):
        run(name)
        torch.cuda.empty_cache()
