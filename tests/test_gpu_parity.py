"""GPU path vs the CPU oracle on seeded inputs, plus size-independent properties
at the BASELINE.json sizes.  All calls go through the public API, which calls
the sm_100a library (include/bzc_b200.h) via ctypes."""

import math

import numpy as np
import pytest
import torch

import bzc_oracle as o

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bz():
    import paper_2406_11209_b200 as m

    assert torch.cuda.is_available()
    return m


def _settings(bz, block, fk, ik, fam="dct", mask_bits=None):
    mask = None if mask_bits is None else bz.PruningMask(tuple(block), mask_bits)
    return bz.CodecSettings(tuple(block), bz.FloatKind(fk), bz.IndexKind(ik),
                            bz.TransformFamily(fam), mask)


def _lowpass(block, k):
    return np.indices(block).sum(axis=0) <= k


def parity(bz, x, block, fk, ik, fam="dct", mask_bits=None, report=None):
    """compress + decompress + ops vs oracle; returns the tie fraction."""
    s = _settings(bz, block, fk, ik, fam, mask_bits)
    os_ = o.Settings(block, fk, ik, fam, mask_bits)
    ca = bz.compress(bz.DenseArray.of(x, bz.FloatKind(fk)), s)
    x64 = o.round_to_kind(x, fk)
    ref = o.compress(x64, os_)
    coeffs = o.coefficients(x64, os_)
    got_n = ca.maxima_f64().cpu().numpy()
    if fk == "f64":
        assert np.all((got_n == ref.maxima) | (np.abs(got_n - ref.maxima) <= 8 * np.spacing(ref.maxima)))
    else:
        assert np.array_equal(got_n, ref.maxima)
    got_i = ca.indices.cpu().numpy()
    ties = o.prune_and_flatten(o.tie_mask(coeffs, ref.maxima, len(block), ik), os_.mask_bits)
    diff = got_i != ref.indices
    assert not (diff & ~ties).any(), int((diff & ~ties).sum())
    # decompress of the REFERENCE's compressed data isolates the decompress kernel
    rc = bz.CompressedArray(x.shape, s, ref.maxima, ref.indices)
    dec = bz.decompress(rc).numpy()
    want = o.decompress(ref)
    span = np.max(np.abs(want))
    assert np.max(np.abs(dec - want)) <= 1e-13 * span
    frac = diff.sum() / max(diff.size, 1)
    if report is not None:
        report.append(frac)
    return ca, ref, frac


@pytest.mark.parametrize("shape,block,fk,ik", [
    ((256, 256, 256), (8, 8, 8), "f32", "i8"),      # C1 at full size
    ((512, 512), (4, 4), "f64", "i16"),              # C2 slab
    ((32, 32, 32, 16), (4, 4, 4, 4), "f32", "i8"),   # C5 slab, full mask
    ((100, 70), (8, 8), "f64", "i16"),
    ((1000,), (8,), "f32", "i16"),
    ((333,), (4,), "f64", "i32"),
    ((40, 33, 20), (4, 4, 4), "f32", "i16"),
])
def test_compress_parity_dct(bz, shape, block, fk, ik):
    rng = np.random.default_rng(hash((shape, block)) % 2**32)
    x = rng.normal(size=shape)
    _, _, frac = parity(bz, x, block, fk, ik)
    print(f"tie fraction {shape} {block}: {frac:.3e}")


@pytest.mark.parametrize("shape,block,fk,ik", [
    ((64, 64, 64), (8, 8, 8), "f32", "i8"),
    ((96, 64), (4, 4), "f64", "i16"),
    ((16, 16, 16, 16), (4, 4, 4, 4), "f32", "i8"),
])
def test_compress_parity_haar(bz, shape, block, fk, ik):
    x = np.random.default_rng(7).uniform(-2, 2, size=shape)
    parity(bz, x, block, fk, ik, fam="haar")


def test_compress_parity_c5_lowpass(bz):
    shape = (32, 32, 32, 16)
    x = o.gradient_array(shape) + 0.01 * np.random.default_rng(7).normal(size=shape)
    ca, ref, _ = parity(bz, x, (4, 4, 4, 4), "f32", "i8", mask_bits=_lowpass((4, 4, 4, 4), 4))
    assert ca.indices.shape[-1] == 66


@pytest.mark.parametrize("fk", ["bf16", "f16"])
def test_compress_parity_narrow_kinds(bz, fk):
    x = np.random.default_rng(3).normal(size=(64, 64, 8))
    parity(bz, x, (8, 8, 8), fk, "i16")


def test_generic_block_shapes(bz):
    rng = np.random.default_rng(11)
    for shape, block in [((12, 9, 16), (4, 2, 8)), ((4, 3, 4, 2, 5), (2, 2, 2, 2, 4)),
                         ((40, 40), (32, 32)), ((9, 7), (1, 1)), ((17,), (2,))]:
        parity(bz, rng.normal(size=shape), block, "f64", "i16")


@pytest.mark.parametrize("shape,block,fk,ik", [
    ((64, 64, 64), (8, 8, 8), "f32", "i8"),
    ((256, 128), (4, 4), "f64", "i16"),
    ((16, 16, 16, 16), (4, 4, 4, 4), "f32", "i8"),
    ((96, 64), (8, 8), "f32", "i32"),
])
def test_fast_and_generic_agree(bz, monkeypatch, shape, block, fk, ik):
    """Fused kernel vs the exact generic kernel on the same data."""
    rng = np.random.default_rng(5)
    x = rng.normal(size=shape)
    s = _settings(bz, block, fk, ik)
    assert bz.is_fast_path(s, shape)
    a = bz.DenseArray.of(x, bz.FloatKind(fk))
    fast = bz.compress(a, s)
    fast_dec = bz.decompress(fast).values
    monkeypatch.setenv("BZC_B200_FORCE_GENERIC", "1")
    generic = bz.compress(a, s)
    gen_dec = bz.decompress(fast).values
    monkeypatch.delenv("BZC_B200_FORCE_GENERIC")
    # compress: maxima and indices identical bits (the factored 8^3 kernel
    # proves or recomputes every block)
    assert torch.equal(fast.maxima, generic.maxima)
    assert torch.equal(fast.indices, generic.indices)
    span = float(gen_dec.abs().max())
    assert float((fast_dec - gen_dec).abs().max()) <= 1e-13 * span
    # the exact fused kernels evaluate the reference's FMA chain: identical bits
    monkeypatch.setenv("BZC_B200_EXACT", "1")
    assert torch.equal(bz.decompress(fast).values, gen_dec)
    exact = bz.compress(a, s)
    assert torch.equal(exact.indices, generic.indices) and torch.equal(exact.maxima, generic.maxima)


# ------------------------------------------------------------- building blocks --
def test_block_unblock_transform_bin(bz):
    rng = np.random.default_rng(1)
    x = rng.normal(size=(19, 13, 10))
    a = bz.DenseArray.of(x)
    b = bz.block(a, (8, 4, 2))
    assert np.array_equal(b.blocks.cpu().numpy(), o.block(x, (8, 4, 2)))
    assert np.array_equal(bz.unblock(b).numpy(), x)
    mats = bz.transforms_for((8, 4, 2), bz.TransformFamily.DCT) if hasattr(bz, "transforms_for") else \
        [bz.make_transform(i, bz.TransformFamily.DCT) for i in (8, 4, 2)]
    c = bz.forward_transform(b, mats)
    want = o.forward_transform(o.block(x, (8, 4, 2)), [m.entries for m in mats])
    assert np.allclose(c.blocks.cpu().numpy(), want, rtol=0, atol=1e-13)
    back = bz.inverse_transform(c, mats)
    assert np.allclose(back.blocks.cpu().numpy(), o.block(x, (8, 4, 2)), atol=1e-13)
    m, idx = bz.bin_coefficients(c, bz.IndexKind.I16, bz.FloatKind.F32)
    rm, ri = o.bin_coefficients(c.blocks.cpu().numpy(), 3, "i16", "f32")
    assert np.array_equal(bz.kinds.widen(m).cpu().numpy(), rm)
    assert np.array_equal(idx.cpu().numpy(), ri)  # same coefficients -> bit-exact
    mask = bz.PruningMask((8, 4, 2), rng.uniform(size=(8, 4, 2)) < 0.4)
    flat = bz.prune_and_flatten(idx, mask)
    assert np.array_equal(flat.cpu().numpy(), o.prune_and_flatten(ri, mask.bits))
    full = bz.unflatten(flat, mask)
    assert np.array_equal(full.cpu().numpy(), o.unflatten(flat.cpu().numpy(), mask.bits))


def test_specified_coefficients_exact(bz):
    rng = np.random.default_rng(2)
    x = rng.normal(size=(32, 32))
    s = _settings(bz, (4, 4), "f32", "i16")
    ca = bz.compress(bz.DenseArray.of(x, bz.FloatKind.F32), s)
    ref = o.Compressed(x.shape, o.Settings((4, 4), "f32", "i16"), ca.maxima_f64().cpu().numpy(),
                       ca.indices.cpu().numpy())
    assert np.array_equal(bz.specified_coefficients(ca).blocks.cpu().numpy(),
                          o.specified_coefficients(ref))


# --------------------------------------------------------------- operators --
@pytest.mark.parametrize("shape,block,fk,ik,mask", [
    ((128, 128, 128), (8, 8, 8), "f32", "i8", None),
    ((1024, 1024), (4, 4), "f64", "i16", None),
    ((32, 32, 32, 16), (4, 4, 4, 4), "f32", "i8", "lowpass"),
    ((50, 37, 21), (8, 8, 8), "f32", "i8", None),
])
def test_ops_parity(bz, shape, block, fk, ik, mask):
    rng = np.random.default_rng(9)
    bits = _lowpass(block, 4) if mask == "lowpass" else None
    s = _settings(bz, block, fk, ik, mask_bits=bits)
    os_ = o.Settings(block, fk, ik, "dct", bits)
    xa = rng.uniform(0, 1, size=shape)
    xb = 0.5 * xa + 0.5 * rng.uniform(0, 1, size=shape)
    ra, rb = o.compress(o.round_to_kind(xa, fk), os_), o.compress(o.round_to_kind(xb, fk), os_)
    a = bz.CompressedArray(shape, s, ra.maxima, ra.indices)
    b = bz.CompressedArray(shape, s, rb.maxima, rb.indices)
    # bit-exact elementwise ops
    for got, want in ((bz.add(a, b), o.add(ra, rb)), (bz.subtract(a, b), o.subtract(ra, rb)),
                      (bz.mul_scalar(a, -0.37), o.mul_scalar(ra, -0.37)),
                      (bz.add_scalar(a, 0.25), o.add_scalar(ra, 0.25)),
                      (bz.negate(a), o.negate(ra))):
        assert np.array_equal(got.maxima_f64().cpu().numpy(), want.maxima)
        assert np.array_equal(got.indices.cpu().numpy(), want.indices)
    # reductions
    pairs = {
        "dot": (bz.dot(a, b), o.dot(ra, rb)),
        "l2": (bz.l2_norm(a), o.l2_norm(ra)),
        "mean": (bz.mean(a), o.mean(ra)),
        "mean_pc": (bz.mean(a, True), o.mean(ra, True)),
        "var": (bz.variance(a), o.variance(ra)),
        "cov": (bz.covariance(a, b), o.covariance(ra, rb)),
        "cos": (bz.cosine_similarity(a, b), o.cosine_similarity(ra, rb)),
        "ssim": (bz.ssim(a, b), o.ssim(ra, rb)),
    }
    for k, (g, w) in pairs.items():
        assert math.isclose(g, w, rel_tol=1e-9, abs_tol=1e-12), (k, g, w)


def test_mixed_index_kinds_reduction(bz):
    rng = np.random.default_rng(4)
    x, y = rng.normal(size=(64, 64)), rng.normal(size=(64, 64))
    s8 = _settings(bz, (8, 8), "f32", "i8")
    s16 = _settings(bz, (8, 8), "f64", "i16")
    a = bz.compress(bz.DenseArray.of(x, bz.FloatKind.F32), s8)
    b = bz.compress(bz.DenseArray.of(y, bz.FloatKind.F64), s16)
    ra = o.Compressed(x.shape, o.Settings((8, 8), "f32", "i8"), a.maxima_f64().cpu().numpy(), a.indices.cpu().numpy())
    rb = o.Compressed(y.shape, o.Settings((8, 8), "f64", "i16"), b.maxima_f64().cpu().numpy(), b.indices.cpu().numpy())
    assert math.isclose(bz.dot(a, b), o.dot(ra, rb), rel_tol=1e-9)
    assert math.isclose(bz.dot(b, a), o.dot(rb, ra), rel_tol=1e-9)
    assert math.isclose(bz.covariance(a, b), o.covariance(ra, rb), rel_tol=1e-9, abs_tol=1e-15)


# ------------------------------------------- full-size properties (BASELINE sizes) --
def _fill(bz, shape, kind, seed, dist=0):
    from paper_2406_11209_b200 import _native

    t = torch.empty(shape, dtype=kind.torch_dtype, device="cuda")
    _native.call("bz_fill_random", t.data_ptr(), kind.code, t.numel(), 0, seed, dist,
                 _native.stream_handle())
    return bz.DenseArray.wrap(t, kind)


def test_c2_full_size_properties(bz):
    """8192^2 f64, 4x4, I16: round-trip error bound, l2 vs dense norm, negate identity."""
    a = _fill(bz, (8192, 8192), bz.FloatKind.F64, 2)
    s = _settings(bz, (4, 4), "f64", "i16")
    ca = bz.compress(a, s)
    out = bz.decompress(ca).values
    err = (out - a.values).abs().reshape(2048, 4, 2048, 4).amax(dim=(1, 3))
    nmax = ca.maxima_f64()
    # per-block bound: sum over coefficients of N/(2r) * max|H| <= N/(2r) * 16
    assert bool((err <= nmax / (2 * 32767) * 16 * (1 + 1e-9)).all())
    l2 = bz.l2_norm(ca)
    dense = float(torch.linalg.vector_norm(out).item())
    assert math.isclose(l2, dense, rel_tol=1e-9)
    assert bz.negate(bz.negate(ca)) == ca
    z = bz.decompress(bz.add(ca, bz.negate(ca))).values
    assert int(torch.count_nonzero(z).item()) == 0


def test_c3_full_size_chain(bz):
    """1024^3 f32, 8^3, I8: mul_scalar(add(a,b), .5) then mean / variance vs dense."""
    s = _settings(bz, (8, 8, 8), "f32", "i8")
    a = bz.compress(_fill(bz, (1024, 1024, 1024), bz.FloatKind.F32, 3), s)
    b = bz.compress(_fill(bz, (1024, 1024, 1024), bz.FloatKind.F32, 4), s)
    t = bz.mul_scalar(bz.add(a, b), 0.5)
    m, v = bz.mean(t), bz.variance(t)
    dense = bz.decompress(t, bz.FloatKind.F32).values
    dm = float(dense.double().mean().item())
    dv = float(dense.double().var(unbiased=False).item())
    assert abs(m - dm) <= 1e-6 * max(1.0, abs(dm))
    assert math.isclose(v, dv, rel_tol=1e-5)
    assert math.isclose(bz.l2_norm(a) ** 2, bz.dot(a, a), rel_tol=1e-9)


def test_partition_invariance_of_random_fill(bz):
    from paper_2406_11209_b200 import _native

    full = torch.empty(1 << 20, dtype=torch.float32, device="cuda")
    part = torch.empty(1 << 19, dtype=torch.float32, device="cuda")
    s = _native.stream_handle()
    _native.call("bz_fill_random", full.data_ptr(), 2, full.numel(), 0, 9, 0, s)
    _native.call("bz_fill_random", part.data_ptr(), 2, part.numel(), 1 << 19, 9, 0, s)
    assert torch.equal(full[1 << 19:], part)


@pytest.mark.parametrize("block,ik,keep", [
    ((8, 8), "i8", 5),          # 5 kept < 16 per chunk: staged path
    ((8, 8), "i16", 37),        # odd kept, chunks span two blocks
    ((4, 4, 4), "i8", 23),      # spanning, int8 masks inside a chunk
    ((8, 8), "i32", 64),
    ((8, 8), "i64", 64),
    ((16, 16), "i16", 256),
])
def test_reductions_mask_and_kinds(bz, block, ik, keep):
    """Streaming reductions over every index kind and chunk/block alignment."""
    rng = np.random.default_rng(11)
    shape = tuple(b * g for b, g in zip(block, (7, 5, 3)[:len(block)]))
    bits = np.zeros(int(np.prod(block)), bool)
    bits[0] = True
    bits[1 + rng.permutation(bits.size - 1)[:keep - 1]] = True
    bits = bits.reshape(block)
    s = _settings(bz, block, "f32", ik, mask_bits=bits)
    os_ = o.Settings(block, "f32", ik, "dct", bits)
    xa = rng.normal(size=shape)
    xb = 0.3 * xa + rng.normal(size=shape)
    ra, rb = o.compress(o.round_to_kind(xa, "f32"), os_), o.compress(o.round_to_kind(xb, "f32"), os_)
    a = bz.CompressedArray(shape, s, ra.maxima, ra.indices)
    b = bz.CompressedArray(shape, s, rb.maxima, rb.indices)
    for k, g, w in (("dot", bz.dot(a, b), o.dot(ra, rb)), ("l2", bz.l2_norm(b), o.l2_norm(rb)),
                    ("cov", bz.covariance(a, b), o.covariance(ra, rb)),
                    ("var", bz.variance(a), o.variance(ra)), ("mean", bz.mean(b), o.mean(rb))):
        assert math.isclose(g, w, rel_tol=1e-9, abs_tol=1e-12), (k, g, w)


def test_dct8_flagged_blocks(bz, monkeypatch):
    """Factored 8^3 compress on blocks that must take the exact fix-up: zero,
    constant (exact ties), tiny/subnormal, NaN, inf, integer-valued data, and
    maxima next to an f32 rounding boundary; bit-identical to the exact path."""
    rng = np.random.default_rng(21)
    x = rng.normal(size=(32, 32, 48)).astype(np.float32).astype(np.float64)
    x[0:8, 0:8, 0:8] = 0.0
    x[0:8, 0:8, 8:16] = 5.0
    x[0:8, 8:16, 0:8] = rng.normal(size=(8, 8, 8)) * 1e-300
    x[8:16, 0:8, 0:8] = np.round(rng.normal(size=(8, 8, 8)) * 4)
    x[8:16, 8:16, 8:16] = rng.normal(size=(8, 8, 8)) * 1e-42  # f32 subnormals
    x[16:24, 0:8, 0:8] = np.nan
    x[16:24, 8:16, 16:24][3, 3, 3] = np.inf
    x[24:32, 24:32, 40:48] = rng.integers(-3, 4, size=(8, 8, 8)) * 0.5
    s = _settings(bz, (8, 8, 8), "f32", "i8")
    a = bz.DenseArray.of(x, bz.FloatKind.F32)
    fast = bz.compress(a, s)
    monkeypatch.setenv("BZC_B200_EXACT", "1")
    exact = bz.compress(a, s)
    monkeypatch.setenv("BZC_B200_FORCE_GENERIC", "1")
    generic = bz.compress(a, s)
    for ref in (exact, generic):  # NaN maxima compare as NaN (sign bit not significant)
        assert np.array_equal(fast.maxima.cpu().numpy(), ref.maxima.cpu().numpy(), equal_nan=True)
        assert torch.equal(fast.indices, ref.indices)
    os_ = o.Settings((8, 8, 8), "f32", "i8", "dct")
    want = o.compress(o.round_to_kind(x, "f32"), os_)
    assert np.array_equal(fast.maxima_f64().cpu().numpy(), want.maxima, equal_nan=True)
    assert np.array_equal(fast.indices.cpu().numpy(), want.indices)


@pytest.mark.parametrize("mask", [None, "lowpass"])
def test_dct4_flagged_blocks(bz, monkeypatch, mask):
    """Factored 4^4 compress (the C5 path) on blocks that need the exact fix-up
    and on a ragged shape: bit-identical to the exact kernels and the oracle."""
    rng = np.random.default_rng(22)
    x = rng.normal(size=(8, 12, 8, 10)).astype(np.float32).astype(np.float64)
    x[0:4, 0:4, 0:4, 0:4] = 0.0
    x[0:4, 0:4, 4:8, 0:4] = 5.0
    x[4:8, 0:4, 0:4, 0:4] = rng.normal(size=(4, 4, 4, 4)) * 1e-42
    x[4:8, 4:8, 0:4, 4:8] = np.round(rng.normal(size=(4, 4, 4, 4)) * 3)
    x[0:4, 8:12, 4:8, 4:8] = np.nan
    x[4:8, 8:12, 4:8, 8] = np.inf
    bits = _lowpass((4, 4, 4, 4), 4) if mask else None
    s = _settings(bz, (4, 4, 4, 4), "f32", "i8", mask_bits=bits)
    a = bz.DenseArray.of(x, bz.FloatKind.F32)
    fast = bz.compress(a, s)
    monkeypatch.setenv("BZC_B200_EXACT", "1")
    exact = bz.compress(a, s)
    monkeypatch.setenv("BZC_B200_FORCE_GENERIC", "1")
    generic = bz.compress(a, s)
    for ref in (exact, generic):  # NaN maxima compare as NaN (sign bit not significant)
        assert np.array_equal(fast.maxima.cpu().numpy(), ref.maxima.cpu().numpy(), equal_nan=True)
        assert torch.equal(fast.indices, ref.indices)
    monkeypatch.delenv("BZC_B200_FORCE_GENERIC")
    monkeypatch.delenv("BZC_B200_EXACT")
    os_ = o.Settings((4, 4, 4, 4), "f32", "i8", "dct", bits)
    want = o.compress(o.round_to_kind(x, "f32"), os_)
    assert np.array_equal(fast.maxima_f64().cpu().numpy(), want.maxima, equal_nan=True)
    assert np.array_equal(fast.indices.cpu().numpy(), want.indices)
    # decompress of finite blocks within the stated tolerance
    dec = bz.decompress(fast).numpy()
    ref = o.decompress(want)
    fin = np.isfinite(ref)
    assert np.array_equal(np.isnan(dec), np.isnan(ref))
    assert np.all(np.abs(dec[fin] - ref[fin]) <= 1e-13 * np.max(np.abs(ref[fin])))


@pytest.mark.parametrize("block,fk,ik,keep", [
    ((8, 8), "f32", "i8", 9),            # tiled add: 8 lanes per block, 4 per lane
    ((8, 8), "f64", "i16", 37),          # 74-byte blocks
    ((16, 16), "f32", "i8", 100),        # 8 lanes x 16
    ((16, 16), "f64", "i8", 200),        # 32 lanes per block
    ((8, 8, 16), "f32", "i16", 300),     # 32 lanes x 16 (600-byte blocks)
    ((8, 8, 16), "f64", "i8", 700),      # > 512 kept: two-pass staged add
    # whole 16-byte chunks, int8 + float32 maxima: the t_hi/t_lo kernel (bz_add8.cu)
    ((8, 8, 8), "f32", "i8", 512),       # C3 / C4: 32 lanes per block
    ((8, 8, 8), "f32", "i8", 256),       # 16 lanes per block
    ((4, 4, 4, 4), "f32", "i8", 64),     # 4 lanes per block
    ((8, 8), "f32", "i8", 16),           # one lane per block
    ((16, 16, 8), "f32", "i8", 1024),    # two chunks per lane
])
def test_elementwise_unaligned_blocks(bz, block, fk, ik, keep):
    """add / subtract / add_scalar / negate on blocks whose kept indices are
    not whole 16-byte vectors (the shared-memory tiled kernels), including
    zero, NaN, tiny and huge blocks; bit-exact with the oracle."""
    rng = np.random.default_rng(keep)
    grid = (5, 3) + (1,) * (len(block) - 2)
    shape = tuple(b * g for b, g in zip(block, grid))
    bits = np.zeros(int(np.prod(block)), bool)
    bits[0] = True
    bits[1 + rng.permutation(bits.size - 1)[:keep - 1]] = True
    bits = bits.reshape(block)
    s = _settings(bz, block, fk, ik, mask_bits=bits)
    os_ = o.Settings(block, fk, ik, "dct", bits)
    xa = rng.normal(size=shape)
    xb = 0.4 * xa + rng.normal(size=shape)
    sl = lambda i: tuple([slice(i * block[0], (i + 1) * block[0])] + [slice(0, b) for b in block[1:]])
    xa[sl(0)] = 0.0
    xb[sl(1)] = np.nan
    xa[sl(2)] *= 1e-300 if fk == "f64" else 1e-30
    xb[sl(3)] *= 1e300 if fk == "f64" else 1e30
    ra, rb = o.compress(o.round_to_kind(xa, fk), os_), o.compress(o.round_to_kind(xb, fk), os_)
    a = bz.CompressedArray(shape, s, ra.maxima, ra.indices)
    b = bz.CompressedArray(shape, s, rb.maxima, rb.indices)
    for got, want in ((bz.add(a, b), o.add(ra, rb)), (bz.subtract(a, b), o.subtract(ra, rb)),
                      (bz.add_scalar(a, 0.25), o.add_scalar(ra, 0.25)),
                      (bz.negate(b), o.negate(rb))):
        assert np.array_equal(got.maxima_f64().cpu().numpy(), want.maxima, equal_nan=True)
        assert np.array_equal(got.indices.cpu().numpy(), want.indices)
    # fused subtract + l2 (the time-series step) over the same blocks; the
    # NaN block makes the full result NaN, so also check the array without it
    assert math.isnan(bz.subtract_l2(a, b)) and math.isnan(o.l2_norm(o.subtract(ra, rb)))
    xb[sl(1)] = rng.normal(size=xb[sl(1)].shape)
    rb = o.compress(o.round_to_kind(xb, fk), os_)
    b = bz.CompressedArray(shape, s, rb.maxima, rb.indices)
    for p_, q_, rp, rq in ((a, b, ra, rb), (b, a, rb, ra)):
        got, want = bz.subtract_l2(p_, q_), o.l2_norm(o.subtract(rp, rq))
        assert math.isclose(got, want, rel_tol=1e-12), (got, want)


@pytest.mark.parametrize("shape,block,mask", [
    ((64, 64, 64), (8, 8, 8), None),
    ((16, 16, 16, 16), (4, 4, 4, 4), "lowpass"),
    ((16, 16, 16, 16), (4, 4, 4, 4), None),
])
def test_negative_dominant_coefficients(bz, shape, block, mask):
    """Blocks whose largest-magnitude coefficient is negative and sits first in
    a lane's maximum chain (the DC term of negative, nearly constant blocks),
    and differences of nearly equal arrays (cancellation: a small negative DC
    dominates).  Guards the compare-select maximum in the factored compress
    kernels and the add kernels."""
    rng = np.random.default_rng(99)
    bits = _lowpass(block, 4) if mask == "lowpass" else None
    x = -(1.0 + 0.01 * rng.normal(size=shape))
    y = x + 1e-4 * rng.normal(size=shape) + 3e-3
    ca, ra, _ = parity(bz, x, block, "f32", "i8", mask_bits=bits)
    cb, rb, _ = parity(bz, y, block, "f32", "i8", mask_bits=bits)
    for got, want in ((bz.subtract(ca, cb), o.subtract(ra, rb)), (bz.add(ca, cb), o.add(ra, rb)),
                      (bz.subtract(cb, ca), o.subtract(rb, ra))):
        assert np.array_equal(got.maxima_f64().cpu().numpy(), want.maxima)
        assert np.array_equal(got.indices.cpu().numpy(), want.indices)


@pytest.mark.parametrize("keep", [1, 3, 9, 15, 17, 31, 47, 66, 95, 127])
def test_add_small_kernel_every_group_width(bz, keep):
    """bz_add_small.cu (int8 / float32 blocks, kept count not a multiple of
    16, one template per ceil(K / 8)): add / subtract / add_scalar /
    subtract+l2 bit-exact with the oracle for K across every lane width,
    over a grid of several tiles with zero, tiny, huge and NaN blocks and
    exact-path (near-half) blocks from nearly equal operands."""
    block = (4, 4, 8)
    rng = np.random.default_rng(1000 + keep)
    grid = (9, 7, 5)  # 315 blocks: several tiles for every K
    shape = tuple(b * g for b, g in zip(block, grid))
    bits = np.zeros(128, bool)
    bits[0] = True
    bits[1 + rng.permutation(127)[:keep - 1]] = True
    bits = bits.reshape(block)
    s = _settings(bz, block, "f32", "i8", mask_bits=bits)
    os_ = o.Settings(block, "f32", "i8", "dct", bits)
    xa = rng.normal(size=shape)
    xb = xa + 1e-3 * rng.normal(size=shape)  # near-cancelling: small coefficients
    xa[:4, :4, :8] = 0.0
    xb[4:8, :4, :8] = np.nan
    xa[8:12, :4, :8] *= 1e-38
    xb[12:16, :4, :8] *= 1e37
    ra, rb = o.compress(o.round_to_kind(xa, "f32"), os_), o.compress(o.round_to_kind(xb, "f32"), os_)
    a = bz.CompressedArray(shape, s, ra.maxima, ra.indices)
    b = bz.CompressedArray(shape, s, rb.maxima, rb.indices)
    for got, want in ((bz.add(a, b), o.add(ra, rb)), (bz.subtract(a, b), o.subtract(ra, rb)),
                      (bz.add_scalar(a, -0.75), o.add_scalar(ra, -0.75))):
        assert np.array_equal(got.maxima_f64().cpu().numpy(), want.maxima, equal_nan=True)
        assert np.array_equal(got.indices.cpu().numpy(), want.indices)
        assert torch.equal(got.dc_plane, got.indices[..., 0])
    assert math.isnan(bz.subtract_l2(a, b))
    xb[4:8, :4, :8] = 0.5
    rb = o.compress(o.round_to_kind(xb, "f32"), os_)
    b = bz.CompressedArray(shape, s, rb.maxima, rb.indices)
    got, want = bz.subtract_l2(b, a), o.l2_norm(o.subtract(rb, ra))
    assert math.isclose(got, want, rel_tol=1e-12), (got, want)


@pytest.mark.parametrize("shape,mask", [
    ((14, 9, 7, 30), None),       # grid (4,3,2,8): TMA box stores + bulk super tiles, ragged edges
    ((14, 9, 7, 30), "lowpass"),
    ((6, 5, 3, 22), "lowpass"),   # grid (2,2,1,6): 24 blocks, TMA stores, bulk super tiles
    ((5, 4, 4, 12), None),        # grid (2,1,1,3): odd last-axis grid -> per-lane row stores
])
def test_dct4_decompress_store_paths(bz, shape, mask):
    """k_dct4_decompress paths: TMA box stores clipped at ragged array edges,
    bulk-copied 8-block super tiles, and per-lane stores; f64 and f32 out,
    1e-13 against the oracle on the reference's compressed data."""
    block = (4, 4, 4, 4)
    bits = _lowpass(block, 4) if mask == "lowpass" else None
    x = np.random.default_rng(sum(shape)).normal(size=shape)
    ca, ref, _ = parity(bz, x, block, "f32", "i8", mask_bits=bits)
    s = _settings(bz, block, "f32", "i8", mask_bits=bits)
    rc = bz.CompressedArray(x.shape, s, ref.maxima, ref.indices)
    want = o.decompress(ref)
    got32 = bz.decompress(rc, bz.FloatKind.F32).numpy().astype(np.float64)
    assert np.max(np.abs(got32 - want)) <= 4e-7 * np.max(np.abs(want))


@pytest.mark.parametrize("shape", [(24, 40, 40), (16, 16, 24), (8, 8, 8)])
def test_dct8_decompress_bulk_tiles(bz, shape):
    """k_dct8_decompress with bulk-copied warp tiles, including an odd block
    count (a last tile of one block) and a single block; f64 and f32 out."""
    block = (8, 8, 8)
    x = np.random.default_rng(sum(shape)).normal(size=shape)
    ca, ref, _ = parity(bz, x, block, "f32", "i8")
    s = _settings(bz, block, "f32", "i8")
    rc = bz.CompressedArray(x.shape, s, ref.maxima, ref.indices)
    want = o.decompress(ref)
    got32 = bz.decompress(rc, bz.FloatKind.F32).numpy().astype(np.float64)
    assert np.max(np.abs(got32 - want)) <= 4e-7 * np.max(np.abs(want))


def _random_compressed(rng, grid, kept, scale=1.0):
    """Synthetic int8 / float32 compressed blocks: indices in [-127, 127]
    with one +-127 per block (a valid binning), float32 maxima."""
    nb = int(np.prod(grid))
    idx = rng.integers(-126, 127, size=(nb, kept), dtype=np.int8)
    pos = rng.integers(0, kept, size=nb)
    idx[np.arange(nb), pos] = np.where(rng.random(nb) < 0.5, -127, 127).astype(np.int8)
    mx = (scale * np.exp(rng.normal(size=nb))).astype(np.float32).astype(np.float64)
    return mx.reshape(grid), idx.reshape(tuple(grid) + (kept,))


@pytest.mark.parametrize("block,keep", [((8, 8, 16), 1024), ((8, 8, 16), 768)])
def test_add8_two_chunks_per_lane(bz, block, keep):
    """bz_add8.cu with blocks of more than 512 kept (two 16-byte chunks per
    lane, 32 lanes per block): add / subtract / add_scalar vs the oracle."""
    rng = np.random.default_rng(17)
    bits = np.zeros(int(np.prod(block)), bool)
    bits[0] = True
    bits[1 + rng.permutation(bits.size - 1)[:keep - 1]] = True
    bits = bits.reshape(block)
    s = _settings(bz, block, "f32", "i8", mask_bits=bits)
    os_ = o.Settings(block, "f32", "i8", "dct", bits)
    grid = (3, 4, 5)
    shape = tuple(b * g for b, g in zip(block, grid))
    ma, ia = _random_compressed(rng, grid, keep)
    mb, ib = _random_compressed(rng, grid, keep, scale=0.5)
    ra, rb = o.Compressed(shape, os_, ma, ia), o.Compressed(shape, os_, mb, ib)
    a = bz.CompressedArray(shape, s, ma.astype(np.float32), ia)
    b = bz.CompressedArray(shape, s, mb.astype(np.float32), ib)
    for got, want in ((bz.add(a, b), o.add(ra, rb)), (bz.subtract(a, b), o.subtract(ra, rb)),
                      (bz.add_scalar(a, 0.25), o.add_scalar(ra, 0.25))):
        assert np.array_equal(got.maxima_f64().cpu().numpy(), want.maxima)
        assert np.array_equal(got.indices.cpu().numpy(), want.indices)
    got, want = bz.subtract_l2(a, b), o.l2_norm(o.subtract(ra, rb))
    assert math.isclose(got, want, rel_tol=1e-12), (got, want)


def test_add8_large_array_group_width(bz):
    """Arrays of >= 2^18 blocks of 512 int8 (the C3 shape class) run add8
    with 16 lanes per block and two chunks per lane: a random sample of
    blocks is checked against the oracle block by block (the operators are
    block-local), and the fused subtract + l2 against l2_norm(subtract)."""
    rng = np.random.default_rng(23)
    block, keep = (8, 8, 8), 512
    grid = (64, 64, 64)  # 262144 blocks
    shape = tuple(b * g for b, g in zip(block, grid))
    s = _settings(bz, block, "f32", "i8")
    ma, ia = _random_compressed(rng, grid, keep)
    mb, ib = _random_compressed(rng, grid, keep, scale=2.0)
    a = bz.CompressedArray(shape, s, ma.astype(np.float32), ia)
    b = bz.CompressedArray(shape, s, mb.astype(np.float32), ib)
    sample = np.sort(rng.choice(int(np.prod(grid)), size=1500, replace=False))
    os_ = o.Settings(block, "f32", "i8")
    sub_shape = (8 * sample.size, 8, 8)
    pick = lambda m, i: (m.reshape(-1)[sample].reshape(-1, 1, 1),
                         i.reshape(-1, keep)[sample].reshape(-1, 1, 1, keep))
    ra = o.Compressed(sub_shape, os_, *pick(ma, ia))
    rb = o.Compressed(sub_shape, os_, *pick(mb, ib))
    for got, want in ((bz.add(a, b), o.add(ra, rb)), (bz.subtract(a, b), o.subtract(ra, rb))):
        gm = got.maxima_f64().cpu().numpy().reshape(-1)[sample]
        gi = got.indices.cpu().numpy().reshape(-1, keep)[sample]
        assert np.array_equal(gm, want.maxima.reshape(-1))
        assert np.array_equal(gi, want.indices.reshape(-1, keep))
    fused, ref = bz.subtract_l2(a, b), bz.l2_norm(bz.subtract(a, b))
    assert math.isclose(fused, ref, rel_tol=1e-12), (fused, ref)


@pytest.mark.parametrize("fk", ["f64", "f32"])
def test_add_rebinning_exact_halves(bz, fk):
    """16-bit rebinning on exact and near rounding halves (k_add's kMagicH
    path hands them to the exact binning): blocks whose sums rebin to
    +-r/2 and (2j+1)/2 positions, ties-to-even as the reference
    (codec.py:272-277, ops.py:178-204); bit-exact with the oracle for add,
    subtract, add_scalar and the fused subtract+l2."""
    rng = np.random.default_rng(11)
    block, grid = (4, 4), (24, 16)
    shape = (block[0] * grid[0], block[1] * grid[1])
    nb = grid[0] * grid[1]
    fmax = 2 * rng.integers(1, 16383, size=nb)
    fa = rng.integers(-1, 2, size=(nb, 16)) * (fmax[:, None] // 2)
    fa[:, 0] = fmax
    fa[:, 5:] = rng.integers(-fmax[:, None] // 2, fmax[:, None] // 2 + 1, size=(nb, 11))
    fb = np.where(rng.random((nb, 16)) < 0.5, 0, rng.integers(-3, 4, size=(nb, 16)))
    fb[:, 0] = 0
    na = rng.choice([1.0, 0.75, 3.0, 2.0 ** -20], size=nb)
    nbm = np.where(rng.random(nb) < 0.5, na, rng.choice([1.0, 0.5, 6.0], size=nb))
    s = _settings(bz, block, fk, "i16")
    os_ = o.Settings(block, fk, "i16", "dct")
    ra = o.Compressed(shape, os_, na.reshape(grid), fa.reshape(grid + (16,)).astype(np.int16))
    rb = o.Compressed(shape, os_, nbm.reshape(grid), fb.reshape(grid + (16,)).astype(np.int16))
    a = bz.CompressedArray(shape, s, ra.maxima, ra.indices)
    b = bz.CompressedArray(shape, s, rb.maxima, rb.indices)
    for got, want in ((bz.add(a, b), o.add(ra, rb)), (bz.subtract(a, b), o.subtract(ra, rb)),
                      (bz.add_scalar(a, 0.5), o.add_scalar(ra, 0.5))):
        assert np.array_equal(got.maxima_f64().cpu().numpy(), want.maxima)
        assert np.array_equal(got.indices.cpu().numpy(), want.indices)
    want_l2 = o.l2_norm(o.subtract(ra, rb))
    assert bz.subtract_l2(a, b) == pytest.approx(want_l2, rel=1e-12)


def test_add8_float32_maximum_edges(bz):
    """add8 (int8 indices, F32 maxima, 8^3 blocks) takes the block maximum
    in float32 (max RN32|c| = RN32 max|c|): exact halves, sums whose maximum
    rounds to an f32 subnormal or overflows (exact path), zero blocks --
    bit-exact with the oracle (ops.py:178-204)."""
    rng = np.random.default_rng(12)
    block, grid = (8, 8, 8), (6, 4, 4)
    shape = tuple(b * g for b, g in zip(block, grid))
    nb, K = int(np.prod(grid)), 512
    fa = rng.integers(-127, 128, size=(nb, K))
    fa[:, 0] = 126
    fa[:, 1] = 63  # 63/126 * 127 = 63.5: an exact half
    fb = np.where(rng.random((nb, K)) < 0.7, 0, rng.integers(-2, 3, size=(nb, K)))
    na = rng.choice([1.0, 0.375, 1e-39, 3e38, 2.0 ** -126], size=nb).astype(np.float32).astype(np.float64)
    nbm = np.where(rng.random(nb) < 0.5, na, 1.0)
    fa[-1] = 0
    fb[-1] = 0  # an all-zero block
    s = _settings(bz, block, "f32", "i8")
    os_ = o.Settings(block, "f32", "i8", "dct")
    ra = o.Compressed(shape, os_, na.reshape(grid), fa.reshape(grid + (K,)).astype(np.int8))
    rb = o.Compressed(shape, os_, nbm.reshape(grid), fb.reshape(grid + (K,)).astype(np.int8))
    a = bz.CompressedArray(shape, s, ra.maxima, ra.indices)
    b = bz.CompressedArray(shape, s, rb.maxima, rb.indices)
    for got, want in ((bz.add(a, b), o.add(ra, rb)), (bz.subtract(a, b), o.subtract(ra, rb))):
        assert np.array_equal(got.maxima_f64().cpu().numpy(), want.maxima)
        assert np.array_equal(got.indices.cpu().numpy(), want.indices)
