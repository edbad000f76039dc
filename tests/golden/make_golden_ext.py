"""Golden vectors for the SURVEY §8f rows, from the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_ext.py

Writes tests/golden/ext.npz: for each case the reference's compressed
arrays (maxima bit patterns, indices), their .bzc streams
(bzc.format.serialize), block means (bzc.ops.block_means), the approximate
Wasserstein distance (bzc.ops.approx_wasserstein, orders 1 / 2 / 3.5) and the
time-series l2 distances of the CLI workflow (cli.py:225-259:
l2_norm(add(s[i+1], negate(s[i])))) -- all computed by the reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("BZC_REFERENCE_SRC", "/root/reference/pkg/src"))

import bzc  # noqa: E402
from bzc import ops as bops  # noqa: E402
from bzc.format import serialize  # noqa: E402
from bzc import metrics as bmetrics  # noqa: E402
from bzc.kinds import FloatKind, IndexKind  # noqa: E402

FK = {k.value: k for k in FloatKind}
IK = {k.value: k for k in IndexKind}

# name, shape, block, float kind, index kind, mask spec, data
CASES = [
    ("f32_i8_3d", (20, 16, 24), (8, 8, 8), "f32", "i8", "full", "normal"),
    ("f64_i16_2d", (33, 20), (4, 4), "f64", "i16", "full", "normal"),
    ("bf16_i16_odd", (12, 12), (4, 4), "bf16", "i16", "full", "normal"),   # 9 blocks: odd
    ("f16_i32_mask", (8, 12, 4), (4, 4, 4), "f16", "i32", "first:21", "uniform"),
    ("f32_i64_1d", (37,), (8,), "f32", "i64", "full", "normal"),
    ("f32_i8_4d_lowpass", (8, 8, 8, 8), (4, 4, 4, 4), "f32", "i8", "lowpass:4", "uniform"),
    ("f32_i8_nan", (16, 16), (8, 8), "f32", "i8", "full", "nan"),
    ("f64_i8_tiny", (8, 8), (2, 2), "f64", "i8", "full", "tiny"),
]


def mask_bits(spec, bshape):
    n = int(np.prod(bshape))
    if spec == "full":
        return np.ones(bshape, dtype=bool)
    kind, _, arg = spec.partition(":")
    if kind == "first":
        bits = np.zeros(n, dtype=bool)
        bits[: int(arg)] = True
        return bits.reshape(bshape)
    if kind == "lowpass":
        return np.indices(bshape).sum(axis=0) <= int(arg)
    raise ValueError(spec)


def data(kind, shape, rng):
    if kind == "normal":
        return rng.normal(size=shape)
    if kind == "uniform":
        return rng.uniform(0, 1, size=shape)
    if kind == "nan":
        x = rng.normal(size=shape)
        x[:8, :8] = np.nan
        return x
    if kind == "tiny":
        return rng.normal(size=shape) * 1e-310
    raise ValueError(kind)


def main():
    rng = np.random.default_rng(2024)
    arrays, table = {}, []
    for name, shape, block, fk, ik, mspec, dkind in CASES:
        bits = mask_bits(mspec, block)
        s = bzc.CodecSettings(block, FK[fk], IK[ik], mask=bzc.PruningMask.from_bits(block, bits))
        xs = [data(dkind, shape, rng) for _ in range(3)]
        arrays[f"{name}/x0"] = xs[0]
        cs = [bzc.compress(bzc.DenseArray.of(x, FK[fk]), s) for x in xs]
        p = f"{name}/"
        arrays[p + "mask"] = bits
        for j, c in enumerate(cs):
            arrays[p + f"max{j}"] = np.asarray(c.maxima_bits())
            arrays[p + f"idx{j}"] = np.asarray(c.indices)
            arrays[p + f"stream{j}"] = np.frombuffer(serialize(c), dtype=np.uint8)
        entry = {"name": name, "shape": list(shape), "block": list(block), "float_kind": fk,
                 "index_kind": ik, "mask": mspec}
        if bits.ravel()[0]:
            arrays[p + "means0"] = np.asarray(bops.block_means(cs[0]), dtype=np.float64)
            w = {}
            for order in (1.0, 2.0, 3.5):
                w[str(order)] = bops.approx_wasserstein(cs[0], cs[1], bops.WassersteinParams(order=order))
            entry["wasserstein"] = w
            entry["timeseries_l2"] = [float(bops.l2_norm(bops.add(cs[i + 1], bops.negate(cs[i]))))
                                      for i in range(2)]
        if dkind != "nan":
            rep = bmetrics.measure_roundtrip(bzc.DenseArray.of(xs[0], FK[fk]), s)
            arrays[p + "bin_bound"] = np.asarray(rep.per_block_bin_bound, dtype=np.float64)
            arrays[p + "loose_linf"] = np.asarray(rep.per_block_loose_linf, dtype=np.float64)
            arrays[p + "l2_coeff"] = np.asarray(rep.per_block_l2_coeff_error, dtype=np.float64)
            arrays[p + "obs_l2_blocks"] = np.asarray(rep.per_block_observed_l2, dtype=np.float64)
            entry["observed_linf"] = rep.observed_linf
            entry["observed_l2"] = rep.observed_l2
            nbytes = len(serialize(cs[0]))
            entry["ratio"] = [bmetrics.compression_ratio(32, s, shape),
                              bmetrics.measured_ratio(32, shape, nbytes), nbytes]
        table.append(entry)
    # Wasserstein on block means that already sum to 1 (no softmax): 1-element blocks
    s1 = bzc.CodecSettings((1, 1), FloatKind.F64, IndexKind.I32)
    pa = rng.uniform(size=(6, 7)); pa /= pa.sum()
    pb = rng.uniform(size=(6, 7)); pb /= pb.sum()
    ca = bzc.compress(bzc.DenseArray.of(pa, FloatKind.F64), s1)
    cb = bzc.compress(bzc.DenseArray.of(pb, FloatKind.F64), s1)
    for j, c in enumerate((ca, cb)):
        arrays[f"normalized/max{j}"] = np.asarray(c.maxima_bits())
        arrays[f"normalized/idx{j}"] = np.asarray(c.indices)
    table.append({"name": "normalized", "shape": [6, 7], "block": [1, 1], "float_kind": "f64",
                  "index_kind": "i32", "mask": "full",
                  "wasserstein": {str(o): bops.approx_wasserstein(ca, cb, bops.WassersteinParams(order=o))
                                  for o in (1.0, 2.0)}})
    np.savez_compressed(os.path.join(HERE, "ext.npz"), **arrays)
    with open(os.path.join(HERE, "ext.json"), "w") as fh:
        json.dump(table, fh, indent=1)
    print(f"{len(table)} cases -> tests/golden/ext.npz, ext.json")


if __name__ == "__main__":
    main()
