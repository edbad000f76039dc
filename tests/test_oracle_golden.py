"""Pin the CPU oracle (oracle/bzc_oracle.py) against the reference's own outputs.

The golden vectors were produced by the real reference (tests/golden/make_golden.py).
Contract: matrices and kind rounding bit-exact; indices bit-exact
except ties; maxima bit-exact for BF16/F16/F32 kinds and within 8 ulps for F64;
decompress within 1e-13 of max|ref|; elementwise ops bit-exact; reductions 1e-9.
"""

import math

import numpy as np
import pytest

import bzc_oracle as o
import golden_io

CASES = golden_io.compress_cases()


def settings_of(case):
    return o.Settings(case["block"], case["float_kind"], case["index_kind"],
                      case["transform"], case["mask"])


def test_matrices_bit_identical():
    arrays, _ = golden_io.load()
    for key, ref in arrays.items():
        if key.startswith("m/"):
            _, fam, size = key.split("/")
            got = o.matrix(int(size), fam)
            assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), key


@pytest.mark.parametrize("kind", ["bf16", "f16", "f32", "f64"])
def test_round_to_kind_bit_identical(kind):
    arrays, _ = golden_io.load()
    got = o.round_to_kind(arrays["k/input"], kind)
    ref = arrays[f"k/{kind}"]
    assert np.array_equal(got, ref, equal_nan=True)
    assert np.array_equal(np.signbit(got), np.signbit(ref))


def test_gradient_bit_identical():
    arrays, _ = golden_io.load()
    assert np.array_equal(o.gradient_array((5, 7, 3)), arrays["g/gradient_5x7x3"])


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_compress_matches_reference(case):
    s = settings_of(case)
    coeffs = o.coefficients(case["input"], s)
    ref_c = case["coeffs"]
    finite = np.isfinite(ref_c)
    assert np.array_equal(finite, np.isfinite(coeffs))
    d = s.ndim
    scale = np.max(np.abs(np.where(finite, ref_c, 0.0)), axis=tuple(range(-d, 0)), keepdims=True)
    limit = np.broadcast_to(1e-14 * scale, ref_c.shape)
    assert np.all(np.abs(coeffs - ref_c)[finite] <= limit[finite] + 1e-300)

    got = o.compress(case["input"], s)
    ref_n = case["maxima"]
    assert got.maxima.shape == ref_n.shape
    both_nan = np.isnan(got.maxima) & np.isnan(ref_n)
    if case["float_kind"] == "f64":
        ok = both_nan | (got.maxima == ref_n) | (golden_io.float_ulps(got.maxima, ref_n, "f64") <= 8)
    else:
        ok = both_nan | (got.maxima == ref_n)
    assert np.all(ok)

    ref_i = case["indices"]
    assert got.indices.dtype == ref_i.dtype and got.indices.shape == ref_i.shape
    ties = o.prune_and_flatten(o.tie_mask(ref_c, ref_n, d, case["index_kind"]), s.mask_bits)
    mismatch = (got.indices != ref_i) & ~ties
    assert not mismatch.any(), int(mismatch.sum())


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_decompress_matches_reference(case):
    s = settings_of(case)
    comp = o.Compressed(case["input"].shape, s, case["maxima"], case["indices"])
    got = o.decompress(comp)
    ref = case["decompressed"]
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    fin = np.isfinite(ref)
    span = np.max(np.abs(ref[fin])) if fin.any() else 0.0
    assert np.all(np.abs(got[fin] - ref[fin]) <= 1e-13 * span + 1e-300)


OPS = golden_io.op_cases()


def _compressed(name):
    case = golden_io.compress_case(name)
    return o.Compressed(case["input"].shape, settings_of(case), case["maxima"], case["indices"])


@pytest.mark.parametrize("case", OPS, ids=[c["name"] for c in OPS])
def test_ops_match_reference(case):
    a, b = _compressed(case["a"]), _compressed(case["b"])
    ref = case["arrays"]
    assert np.array_equal(o.negate(a).indices, ref["negate_idx"])
    for tag, out in (("add", o.add(a, b)), ("sub", o.subtract(a, b)), ("addself", o.add(a, a))):
        assert np.array_equal(out.maxima, ref[f"{tag}_max"], equal_nan=True), tag
        assert np.array_equal(out.indices, ref[f"{tag}_idx"]), tag
    for j, x in enumerate(case["scalars"]):
        m = o.mul_scalar(a, x)
        assert np.array_equal(m.maxima, ref[f"mul{j}_max"], equal_nan=True)
        assert np.array_equal(m.indices, ref[f"mul{j}_idx"])
    if "addscalar_max" in ref:
        asc = o.add_scalar(a, 0.75)
        assert np.array_equal(asc.maxima, ref["addscalar_max"])
        assert np.array_equal(asc.indices, ref["addscalar_idx"])
    res = case["results"]
    got = {
        "dot": o.dot(a, b), "dot_self": o.dot(a, a), "l2_a": o.l2_norm(a),
        "l2_b": o.l2_norm(b), "cos": o.cosine_similarity(a, b),
    }
    if "mean_a" in res:
        lum, con, st = o.ssim_components(a, b)
        got.update({
            "mean_a": o.mean(a), "mean_a_pc": o.mean(a, True), "cov": o.covariance(a, b),
            "var_a": o.variance(a), "var_b": o.variance(b), "ssim_l": lum, "ssim_c": con,
            "ssim_s": st, "ssim": o.ssim(a, b), "ssim_self": o.ssim(a, a),
        })
    for k, v in got.items():
        assert math.isclose(v, res[k], rel_tol=1e-9, abs_tol=1e-12), (k, v, res[k])
