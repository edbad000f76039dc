"""The DC plane: every producer's dc[b] equals indices[b][0], and mean read
from the plane equals mean from the stride-K gather (the
reference's _first_coefficients, ops.py:166-175, and mean, ops.py:244-257)
to 1e-12 relative -- the same per-block arithmetic, summed in another order.

Producers covered: the factored 8^3 / 4^4 compress kernels (fix-up blocks
included), the exact fused 2-D kernel (plane by gather), the generic
kernel, add / subtract / add_scalar (int8 kernel and the general ones),
mul_scalar with x > 0 (aliased), x < 0, 0 and NaN, and negate.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bz():
    import paper_2406_11209_b200 as m

    assert torch.cuda.is_available()
    return m


def _plane_ok(a):
    assert a.dc_plane is not None
    assert a.dc_plane.shape == a.maxima.shape
    assert torch.equal(a.dc_plane, a.indices[..., 0])


def _strip(bz, a):
    """The same array without its plane (mean falls back to the gather)."""
    return bz.CompressedArray(a.original_shape, a.settings, a.maxima, a.indices, _trusted=True)


def _mean_both(bz, a):
    from paper_2406_11209_b200 import ops

    r1 = ops.moments_record(a, dc_only=1).cpu().numpy()
    r0 = ops.moments_record(_strip(bz, a), dc_only=1).cpu().numpy()
    assert r1[0] == r0[0]
    np.testing.assert_allclose(r1[1], r0[1], rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(r1[4], r0[4], rtol=1e-10, atol=1e-300)
    for pc in (False, True):
        m1, m0 = bz.mean(a, padding_corrected=pc), bz.mean(_strip(bz, a), padding_corrected=pc)
        assert (math.isnan(m1) and math.isnan(m0)) or m1 == pytest.approx(m0, rel=1e-12, abs=1e-300)


def _f32(bz, x):
    return bz.DenseArray(x.shape, bz.FloatKind.F32, x.astype(np.float32))


CASES = [
    # shape, block, float kind, index kind, low-pass order (None = full)
    ((40, 64, 48), (8, 8, 8), "f32", "i8", None),         # dct8 (partial blocks)
    ((16, 16, 16, 32), (4, 4, 4, 4), "f32", "i8", 4),     # dct4 low-pass (TMA tiles)
    ((12, 8, 8, 12), (4, 4, 4, 4), "f32", "i8", 4),       # dct4, non-TMA shape
    ((256, 192), (4, 4), "f64", "i16", None),             # exact fused 2-D (+ gather)
    ((24, 20, 12), (4, 4, 4), "f64", "i32", None),        # generic / other fused
    ((64, 48), (8, 8), "f32", "i16", 3),                  # pruned 2-D mask keeping DC
    # float64 maxima over >= 4096 blocks: the bulk-copied plane kernel
    # (69077 / 8385 blocks: ragged multi-stage CTA ranges plus a tail < 16)
    ((4 * 67, 4 * 1031), (4, 4), "f64", "i16", None),
    ((4 * 65, 4 * 129), (4, 4), "f64", "i32", None),
]


def _settings(bz, block, fk, ik, lp):
    mask = None
    if lp is not None:
        mask = bz.PruningMask(block, np.indices(block).sum(axis=0) <= lp)
    return bz.CodecSettings(block, bz.FloatKind(fk), bz.IndexKind(ik), mask=mask)


@pytest.mark.parametrize("shape,block,fk,ik,lp", CASES)
def test_producers_write_the_plane(bz, rng, shape, block, fk, ik, lp):
    s = _settings(bz, block, fk, ik, lp)
    x = rng.normal(size=shape)
    y = rng.normal(size=shape) * 3.0
    kind = bz.FloatKind(fk)
    cx = bz.compress(bz.DenseArray(shape, kind, x.astype(np.float32 if fk == "f32" else np.float64)), s)
    cy = bz.compress(bz.DenseArray(shape, kind, y.astype(np.float32 if fk == "f32" else np.float64)), s)
    _plane_ok(cx)
    _plane_ok(cy)
    for r in (bz.add(cx, cy), bz.subtract(cx, cy), bz.add_scalar(cx, 0.75), bz.negate(cx),
              bz.mul_scalar(cx, 0.5), bz.mul_scalar(cx, -2.0), bz.mul_scalar(cx, 0.0),
              bz.mul_scalar(cx, float("nan"))):
        _plane_ok(r)
        _mean_both(bz, r)
    _mean_both(bz, cx)
    assert bz.mul_scalar(cx, 0.5).dc_plane.data_ptr() == cx.dc_plane.data_ptr()  # aliased


def test_flagged_blocks_keep_the_plane(bz):
    """Zero / constant / tiny / huge blocks go through the exact fix-up
    kernels; their plane entries must follow."""
    s = bz.CodecSettings((8, 8, 8), bz.FloatKind.F32, bz.IndexKind.I8)
    x = np.random.default_rng(3).normal(size=(32, 32, 32)).astype(np.float32)
    x[:8, :8, :8] = 0.0
    x[8:16, :8, :8] = 5.0
    x[16:24, :8, :8] *= 1e-40
    x[24:32, :8, :8] *= 1e37
    c = bz.compress(_f32(bz, x), s)
    _plane_ok(c)
    _mean_both(bz, c)
    s4 = bz.CodecSettings((4, 4, 4, 4), bz.FloatKind.F32, bz.IndexKind.I8,
                          mask=bz.PruningMask((4, 4, 4, 4),
                                              np.indices((4, 4, 4, 4)).sum(axis=0) <= 4))
    x4 = np.random.default_rng(4).normal(size=(16, 16, 16, 64)).astype(np.float32)
    x4[:4, :4, :4, :4] = 0.0
    x4[4:8, :4, :4, :4] = -3.0
    x4[8:12, :4, :4, :4] *= 1e-41
    c4 = bz.compress(_f32(bz, x4), s4)
    _plane_ok(c4)
    _mean_both(bz, c4)


def test_add8_exact_blocks_keep_the_plane(bz):
    """Blocks the int8 add sends through its exact per-block path."""
    s = bz.CodecSettings((8, 8, 8), bz.FloatKind.F32, bz.IndexKind.I8)
    rng = np.random.default_rng(5)
    x = rng.normal(size=(32, 32, 32)).astype(np.float32)
    y = -x.copy()
    y[8:, :, :] = rng.normal(size=(24, 32, 32)).astype(np.float32)
    x[16:24] *= 1e-39
    cx, cy = bz.compress(_f32(bz, x), s), bz.compress(_f32(bz, y), s)
    for r in (bz.add(cx, cy), bz.subtract(cx, cy), bz.add_scalar(cx, 1e-30)):
        _plane_ok(r)
        _mean_both(bz, r)


def test_no_plane_without_first_coefficient(bz, rng):
    bits = np.ones((4, 4), dtype=bool)
    bits[0, 0] = False
    s = bz.CodecSettings((4, 4), bz.FloatKind.F64, bz.IndexKind.I16,
                         mask=bz.PruningMask.from_bits((4, 4), bits))
    c = bz.compress(bz.DenseArray.of(rng.normal(size=(16, 16))), s)
    assert c.dc_plane is None
    assert bz.add(c, c).dc_plane is None


def test_mean_plane_c3_size(bz):
    """BASELINE C3 shape: mean of the chain result through the plane equals
    the gather, and the plane equals indices[..., 0] everywhere."""
    from paper_2406_11209_b200 import _native

    s = bz.CodecSettings((8, 8, 8), bz.FloatKind.F32, bz.IndexKind.I8)
    shape = (1024, 1024, 1024)

    def field(seed):
        t = torch.empty(shape, dtype=torch.float32, device="cuda")
        _native.call("bz_fill_random", t.data_ptr(), bz.FloatKind.F32.code, t.numel(), 0, seed,
                     0, _native.stream_handle())
        return bz.DenseArray.wrap(t, bz.FloatKind.F32)

    cx = bz.compress(field(2), s)
    cy = bz.compress(field(3), s)
    t = bz.mul_scalar(bz.add(cx, cy), 0.5)
    _plane_ok(cx)
    _plane_ok(t)
    _mean_both(bz, t)


@pytest.mark.parametrize("case", [((40, 64, 48), (8, 8, 8), "f32", "i8"),
                                  ((64, 96), (4, 4), "f64", "i16"),
                                  ((16, 16, 16, 32), (4, 4, 4, 4), "f32", "i8")])
def test_block_means_and_wasserstein_from_plane(bz, case):
    """block_means / approx_wasserstein read the DC plane when the array has
    one (bz_block_means_dc, bz_approx_wasserstein_dc): the same bits as the
    K-strided gather of indices[..., 0] (ops.py:166-175, 355-384)."""
    shape, block, fk, ik = case
    rng = np.random.default_rng(7)
    s = bz.CodecSettings(block, bz.FloatKind(fk), bz.IndexKind(ik))
    dt = np.float32 if fk == "f32" else np.float64
    xs = [rng.normal(size=shape).astype(dt) for _ in range(2)]
    a, b = (bz.compress(bz.DenseArray(shape, bz.FloatKind(fk), x), s) for x in xs)
    _plane_ok(a)
    _plane_ok(b)
    assert torch.equal(bz.block_means(a), bz.block_means(_strip(bz, a)))
    for order in (1.0, 2.0, 1.5):
        p = bz.ops.WassersteinParams(order=order)
        w_plane = bz.approx_wasserstein(a, b, p)
        assert w_plane == bz.approx_wasserstein(_strip(bz, a), _strip(bz, b), p)
        assert w_plane == bz.approx_wasserstein(a, _strip(bz, b), p)
