"""Generate golden vectors from the REAL reference package (bzc).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``bzc`` from ``/root/reference/pkg/src`` (or $BZC_REFERENCE_SRC),
runs the reference's own compress / decompress / operator code on seeded
inputs, and writes ``tests/golden/golden.npz`` (inputs + reference outputs)
plus ``tests/golden/cases.json`` (the case table).  The fixtures are
committed; the GPU box never needs the reference itself.

Cases cover the reference's own known-answer tests (pkg/tests/test_codec.py,
test_kinds.py, test_ops.py) and small instances of every BASELINE config
(C1: 3-D f32 8^3 I8; C2: 2-D f64 4^2 I16; C3/C4: 3-D f32 8^3 I8 chains;
C5: 4-D f32 4^4 I8 low-pass mask).
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
from bzc.arrays import block as bblock  # noqa: E402
from bzc.kinds import FloatKind, IndexKind  # noqa: E402
from bzc.transforms import TransformFamily  # noqa: E402

FK = {k.value: k for k in FloatKind}
IK = {k.value: k for k in IndexKind}
TF = {"dct": TransformFamily.DCT, "haar": TransformFamily.HAAR}


def mask_bits(spec: str, bshape):
    n = int(np.prod(bshape))
    if spec == "full":
        return np.ones(bshape, dtype=bool)
    kind, _, arg = spec.partition(":")
    if kind == "first":
        bits = np.zeros(n, dtype=bool)
        bits[: int(arg)] = True
        return bits.reshape(bshape)
    if kind == "lowpass":  # keep positions whose index sum <= arg
        idx = np.indices(bshape).sum(axis=0)
        return idx <= int(arg)
    if kind == "corner":  # Blaz corner drop on 8x8 (test_codec.py:103-114)
        bits = np.ones(bshape, dtype=bool)
        bits[2:, 2:] = False
        return bits
    if kind == "nofirst":
        bits = np.ones(n, dtype=bool)
        bits[0] = False
        return bits.reshape(bshape)
    if kind == "none":
        return np.zeros(bshape, dtype=bool)
    raise ValueError(spec)


def make_input(gen: str, shape, seed: int):
    rng = np.random.default_rng(seed)
    if gen == "normal":
        return rng.normal(size=shape)
    if gen == "uniform":
        return rng.uniform(0, 1, shape)
    if gen == "uniform_pm":
        return rng.uniform(-3, 3, shape)
    if gen == "gradient":
        return bzc.gradient_array(shape).values.copy()
    if gen == "gradient_noise":
        return bzc.gradient_array(shape).values + 0.01 * rng.normal(size=shape)
    if gen.startswith("const:"):
        return np.full(shape, float(gen.split(":")[1]))
    if gen == "zeros":
        return np.zeros(shape)
    if gen == "wide":  # many binades, exercises subnormal/huge maxima
        return rng.normal(size=shape) * 10.0 ** rng.integers(-30, 30, size=shape)
    if gen == "special":
        x = rng.normal(size=shape).ravel()
        x[::7] = 0.0
        if x.size > 3:
            x[1] = np.nan
        if x.size > 11:
            x[-2] = np.inf
        return x.reshape(shape)
    if gen == "tiny":
        return rng.normal(size=shape) * 1e-42
    raise ValueError(gen)


# (name, shape, block, float kind, index kind, transform, mask, input gen, seed, input kind)
COMPRESS_CASES = [
    ("const5_8x8", (8, 8), (8, 8), "f64", "i16", "dct", "full", "const:5.0", 0, "f64"),
    ("zeros_8x8_4x4", (8, 8), (4, 4), "f64", "i16", "dct", "full", "zeros", 0, "f64"),
    ("impulse16_1d", (4,), (4,), "f64", "i8", "dct", "full", "const:0", 0, "f64"),
    ("c1_small", (32, 32, 32), (8, 8, 8), "f32", "i8", "dct", "full", "normal", 0, "f32"),
    ("c1_padded", (19, 21, 13), (8, 8, 8), "f32", "i8", "dct", "full", "normal", 1, "f32"),
    ("c2_small", (64, 64), (4, 4), "f64", "i16", "dct", "full", "normal", 2, "f64"),
    ("c2_padded", (37, 50), (4, 4), "f64", "i16", "dct", "full", "normal", 3, "f64"),
    ("c4_uniform", (16, 16, 16), (8, 8, 8), "f32", "i8", "dct", "full", "uniform", 5, "f32"),
    ("c5_small", (8, 8, 8, 8), (4, 4, 4, 4), "f32", "i8", "dct", "lowpass:4", "gradient_noise", 7, "f32"),
    ("c5_padded", (6, 5, 7, 9), (4, 4, 4, 4), "f32", "i8", "dct", "lowpass:4", "normal", 8, "f32"),
    ("haar_3d", (12, 9, 16), (4, 2, 8), "f32", "i16", "haar", "full", "normal", 9, "f32"),
    ("haar_2d_i32", (20, 24), (8, 8), "f64", "i32", "haar", "full", "uniform_pm", 10, "f64"),
    ("bf16_kind", (16, 16), (4, 4), "bf16", "i8", "dct", "full", "normal", 11, "f64"),
    ("f16_kind", (16, 16), (4, 4), "f16", "i16", "dct", "full", "normal", 12, "f64"),
    ("f32_from_f64", (24, 24), (8, 8), "f32", "i16", "dct", "full", "normal", 13, "f64"),
    ("i64_kind", (16, 8), (4, 8), "f64", "i64", "dct", "full", "normal", 14, "f64"),
    ("corner_mask", (16, 16), (8, 8), "f64", "i16", "dct", "corner", "uniform", 15, "f64"),
    ("first6_mask", (8, 8), (4, 4), "f64", "i16", "dct", "first:6", "uniform", 16, "f64"),
    ("empty_mask", (8, 8), (4, 4), "f64", "i16", "dct", "none", "uniform", 17, "f64"),
    ("unit_blocks", (9, 7), (1, 1), "f64", "i16", "dct", "full", "normal", 18, "f64"),
    ("one_d_16", (37,), (16,), "f32", "i8", "dct", "full", "normal", 19, "f32"),
    ("five_d", (4, 3, 4, 2, 5), (2, 2, 2, 2, 4), "f64", "i16", "dct", "full", "normal", 20, "f64"),
    ("big_block", (40, 40), (32, 32), "f64", "i16", "dct", "full", "normal", 21, "f64"),
    ("wide_range", (16, 16), (4, 4), "f32", "i16", "dct", "full", "wide", 22, "f64"),
    ("special_vals", (16, 16), (4, 4), "f32", "i8", "dct", "full", "special", 23, "f64"),
    ("tiny_vals", (8, 8), (4, 4), "f32", "i16", "dct", "full", "tiny", 24, "f64"),
    ("gradient_16", (16, 16), (4, 4), "f64", "i16", "dct", "full", "gradient", 0, "f64"),
    ("c3_like_8x8_f16in", (16, 8, 8), (8, 8, 8), "f32", "i8", "dct", "full", "normal", 25, "f16"),
]

# (name, a case, b case, scalars for mul_scalar)
OP_CASES = [
    ("ops_c2", "c2_small", "c2_padded_pair", [2.5, -0.251, 0.0, 1e6, -1.0, 1.0]),
    ("ops_c1", "c1_small", "c1_small_pair", [0.5, -3.7]),
    ("ops_c4", "c4_uniform", "c4_uniform_pair", [0.5]),
    ("ops_c5", "c5_small", "c5_small_pair", [0.5, -2.0]),
    ("ops_pad", "c1_padded", "c1_padded_pair", [1.5]),
    ("ops_haar", "haar_3d", "haar_3d_pair", [2.0]),
    ("ops_kinds", "bf16_kind", "bf16_kind_pair", [3.0, -1e-3]),
]


def main():
    arrays: dict[str, np.ndarray] = {}
    table = {"compress": [], "ops": []}
    compressed = {}

    def run_compress(name, shape, bshape, fk, ik, tf, mspec, gen, seed, in_kind):
        raw = make_input(gen, shape, seed)
        if gen == "const:0":
            raw = np.array([1.0, 0.0, 0.0, 0.0]) * 16.0 / 2.0  # DC=16 after 4-pt DCT
        a = bzc.DenseArray.of(raw, FK[in_kind])
        bits = mask_bits(mspec, bshape)
        settings = bzc.CodecSettings(bshape, FK[fk], IK[ik], TF[tf],
                                     bzc.PruningMask(bshape, bits))
        ca = bzc.compress(a, settings)
        lowered = bzc.convert_precision(a, FK[fk])
        coeffs = bzc.forward_transform(bblock(lowered, bshape), settings.matrices()).blocks
        dec = bzc.decompress(ca).values
        p = f"c/{name}/"
        arrays[p + "input"] = a.values
        arrays[p + "mask"] = bits
        arrays[p + "maxima"] = ca.maxima_f64()
        arrays[p + "indices"] = ca.indices
        arrays[p + "coeffs"] = coeffs
        arrays[p + "decompressed"] = dec
        table["compress"].append(dict(name=name, shape=list(shape), block=list(bshape),
                                      float_kind=fk, index_kind=ik, transform=tf,
                                      mask=mspec, gen=gen, seed=seed, input_kind=in_kind))
        compressed[name] = ca

    for case in COMPRESS_CASES:
        run_compress(*case)
    # second operands for the op cases: same settings, different seed
    for opname, an, bn, _ in OP_CASES:
        base = next(c for c in COMPRESS_CASES if c[0] == an)
        seed = base[8] + 1000
        run_compress(bn, *base[1:8], seed, base[9])

    for opname, an, bn, scalars in OP_CASES:
        a, b = compressed[an], compressed[bn]
        p = f"o/{opname}/"
        out = {}
        out["negate_idx"] = bops.negate(a).indices
        s = bops.add(a, b)
        out["add_max"], out["add_idx"] = s.maxima_f64(), s.indices
        d = bops.add(a, bops.negate(b))
        out["sub_max"], out["sub_idx"] = d.maxima_f64(), d.indices
        aa = bops.add(a, a)
        out["addself_max"], out["addself_idx"] = aa.maxima_f64(), aa.indices
        for j, x in enumerate(scalars):
            m = bops.mul_scalar(a, x)
            out[f"mul{j}_max"], out[f"mul{j}_idx"] = m.maxima_f64(), m.indices
        scal = {}
        scal["dot"] = bops.dot(a, b)
        scal["dot_self"] = bops.dot(a, a)
        scal["l2_a"] = bops.l2_norm(a)
        scal["l2_b"] = bops.l2_norm(b)
        if a.settings.mask.keeps_first:
            scal["mean_a"] = bops.mean(a)
            scal["mean_a_pc"] = bops.mean(a, padding_corrected=True)
            scal["cov"] = bops.covariance(a, b)
            scal["var_a"] = bops.variance(a)
            scal["var_b"] = bops.variance(b)
            lum, con, st = bops.ssim_components(a, b)
            scal["ssim_l"], scal["ssim_c"], scal["ssim_s"] = lum, con, st
            scal["ssim"] = bops.ssim(a, b)
            scal["ssim_self"] = bops.ssim(a, a)
            asc = bops.add_scalar(a, 0.75)
            out["addscalar_max"], out["addscalar_idx"] = asc.maxima_f64(), asc.indices
        scal["cos"] = bops.cosine_similarity(a, b)
        for k, v in out.items():
            arrays[p + k] = v
        table["ops"].append(dict(name=opname, a=an, b=bn, scalars=scalars,
                                 results={k: float(v) for k, v in scal.items()}))

    # kind rounding goldens (test_kinds.py:58-113)
    rng = np.random.default_rng(20240817)
    xs = np.concatenate([
        rng.uniform(-1e4, 1e4, 200),
        rng.uniform(-1, 1, 200) * 10.0 ** rng.integers(-45, 39, 200),
        rng.uniform(-1, 1, 100) * 2.0 ** rng.integers(-30, -10, 100),
        np.array([1 / 3, 65519.99, 65520.0, 70000.0, -70000.0, 65504.0, 0.0, -0.0,
                  np.inf, -np.inf, np.nan, 3.4028235677973366e38, 1e-46, 1.4e-45]),
    ])
    arrays["k/input"] = xs
    from bzc.kinds import round_to_kind
    for k in FloatKind:
        arrays[f"k/{k.value}"] = round_to_kind(xs, k)
    arrays["g/gradient_5x7x3"] = bzc.gradient_array((5, 7, 3)).values
    for size in (1, 2, 4, 8, 16, 32):
        for fam in ("dct", "haar"):
            arrays[f"m/{fam}/{size}"] = bzc.make_transform(size, TF[fam]).entries

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "cases.json"), "w") as fh:
        json.dump(table, fh, indent=1)
    size = os.path.getsize(os.path.join(HERE, "golden.npz"))
    print(f"wrote {len(arrays)} arrays, {size / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
