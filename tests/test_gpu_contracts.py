"""The reference's error and edge contracts, through the GPU path.

Mirrors pkg/tests/test_ops.py (SettingsMismatch :115-121, mixed float kinds
:125-130, MaskExcludesMeanCoefficient :156-162 / :264-270 / :444-450,
all-false masks :319-325, ZeroNormOperand :345-347, negative SSIM base with a
fractional weight :377-382) and arrays.py:81-86 (a DenseArray whose values
are not representable raises ValueError), plus the library contracts the
advisor asked for: large blocks in add (I64 8x8x8), huge maxima in the
reductions, mismatched C-ABI layouts, concurrent reductions from several
threads, and a workspace that survives a failed launch.
"""

import ctypes
import math
import threading

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


@pytest.fixture(scope="module")
def S(bz):
    return {
        "S44": bz.CodecSettings((4, 4), bz.FloatKind.F64, bz.IndexKind.I16),
        "S44_I32": bz.CodecSettings((4, 4), bz.FloatKind.F64, bz.IndexKind.I32),
        "S88": bz.CodecSettings((8, 8), bz.FloatKind.F64, bz.IndexKind.I16),
    }


def comp(bz, values, settings):
    return bz.compress(bz.DenseArray.of(np.asarray(values, dtype=np.float64)), settings)


def _no_first(bz, shape, fk=None):
    bits = np.ones(shape, dtype=bool)
    bits.reshape(-1)[0] = False
    return bz.CodecSettings(shape, fk or bz.FloatKind.F64,
                            mask=bz.PruningMask.from_bits(shape, bits))


def test_add_requires_compatible_operands(bz, S, rng):
    a = comp(bz, rng.uniform(size=(16, 16)), S["S44"])
    b = comp(bz, rng.uniform(size=(16, 16)),
             bz.CodecSettings((4, 4), bz.FloatKind.F64, bz.IndexKind.I8))
    with pytest.raises(bz.errors.SettingsMismatch):
        bz.add(a, b)
    c = comp(bz, rng.uniform(size=(8, 8)), S["S88"])
    with pytest.raises(bz.errors.SettingsMismatch):
        bz.add(a, c)
    with pytest.raises(bz.errors.SettingsMismatch):
        bz.dot(a, c)
    with pytest.raises(bz.errors.SettingsMismatch):
        bz.covariance(a, c)


def test_add_allows_different_float_kinds(bz, rng):
    x = rng.uniform(size=(8, 8))
    a = comp(bz, x, bz.CodecSettings((4, 4), bz.FloatKind.F64, bz.IndexKind.I16))
    b = comp(bz, x, bz.CodecSettings((4, 4), bz.FloatKind.F32, bz.IndexKind.I16))
    out = bz.add(a, b)
    assert out.settings.float_kind is bz.FloatKind.F64
    # bit-exact with the oracle's add under a's kinds (ops.py:200-204)
    ra = o.Compressed((8, 8), o.Settings((4, 4), "f64", "i16"), a.maxima_f64().cpu().numpy(),
                      a.indices.cpu().numpy())
    rb = o.Compressed((8, 8), o.Settings((4, 4), "f32", "i16"), b.maxima_f64().cpu().numpy(),
                      b.indices.cpu().numpy())
    want = o.add(ra, rb)
    assert np.array_equal(out.maxima_f64().cpu().numpy(), want.maxima)
    assert np.array_equal(out.indices.cpu().numpy(), want.indices)
    # and the other way round: F32 result
    out2 = bz.add(b, a)
    assert out2.settings.float_kind is bz.FloatKind.F32
    want2 = o.add(rb, ra)
    assert np.array_equal(out2.maxima_f64().cpu().numpy(), want2.maxima)
    assert np.array_equal(out2.indices.cpu().numpy(), want2.indices)


def test_mask_excludes_mean_coefficient(bz, rng):
    a = comp(bz, rng.uniform(size=(8, 8)), _no_first(bz, (4, 4)))
    for fn in (lambda: bz.add_scalar(a, 1.0), lambda: bz.mean(a), lambda: bz.variance(a),
               lambda: bz.covariance(a, a), lambda: bz.ssim(a, a),
               lambda: bz.block_means(a)):
        with pytest.raises(bz.errors.MaskExcludesMeanCoefficient):
            fn()
    w = comp(bz, rng.uniform(size=16), _no_first(bz, (4,)))
    with pytest.raises(bz.errors.MaskExcludesMeanCoefficient):
        bz.approx_wasserstein(w, w, bz.WassersteinParams())
    # the reductions that do not need it still work (and match the oracle)
    ra = o.Compressed((8, 8), o.Settings((4, 4), "f64", "i16", "dct",
                                         np.array(a.settings.mask.bits)),
                      a.maxima_f64().cpu().numpy(), a.indices.cpu().numpy())
    assert math.isclose(bz.l2_norm(a), o.l2_norm(ra), rel_tol=1e-12)
    assert math.isclose(bz.dot(a, a), o.dot(ra, ra), rel_tol=1e-12)


def test_reductions_with_all_false_mask(bz, rng):
    mask = bz.PruningMask.from_bits((4, 4), np.zeros(16, dtype=bool))
    s = bz.CodecSettings((4, 4), bz.FloatKind.F64, bz.IndexKind.I16, mask=mask)
    a = comp(bz, rng.uniform(size=(8, 8)), s)
    assert a.indices.shape == (2, 2, 0)
    assert bz.l2_norm(a) == 0.0
    assert bz.dot(a, a) == 0.0
    assert bz.subtract_l2(a, a) == 0.0  # no kept coefficient: the empty-case store
    with pytest.raises(bz.errors.ZeroNormOperand):
        bz.cosine_similarity(a, a)
    assert int(torch.count_nonzero(bz.decompress(a).values).item()) == 0


def test_cosine_similarity_zero_norm(bz, S, rng):
    a = comp(bz, rng.uniform(-1, 1, (16, 16)), S["S44"])
    z = comp(bz, np.zeros((16, 16)), S["S44"])
    with pytest.raises(bz.errors.ZeroNormOperand):
        bz.cosine_similarity(a, z)
    with pytest.raises(bz.errors.ZeroNormOperand):
        bz.cosine_similarity(z, a)
    assert bz.l2_norm(z) == 0.0


def test_ssim_negative_base_fractional_weight(bz, S, rng):
    a = comp(bz, rng.uniform(0, 1, (16, 16)), S["S44"])
    b = bz.negate(a)
    with pytest.raises(bz.errors.NegativeBaseWithFractionalWeight):
        bz.ssim(a, b, bz.SsimParams(structure_weight=0.5))
    assert np.isfinite(bz.ssim(a, b, bz.SsimParams()))
    with pytest.raises(ValueError):
        bz.SsimParams(luminance_stabilizer=-1.0)


def test_dense_array_not_representable(bz):
    with pytest.raises(ValueError):
        bz.DenseArray((3,), bz.FloatKind.F32, np.array([0.1, 0.2, 0.3]))
    with pytest.raises(ValueError):
        bz.DenseArray((2,), bz.FloatKind.F16, torch.tensor([1.0, 1e-9], dtype=torch.float64))
    ok = bz.DenseArray((2,), bz.FloatKind.F32, np.array([0.5, 0.25]))
    assert ok.kind is bz.FloatKind.F32


def test_reference_edge_values(bz, S, rng):
    """test_ops.py: constants, zeros, self-similarity (the GPU path)."""
    assert bz.covariance(comp(bz, np.full((8, 8), 3.0), S["S88"]),
                         comp(bz, np.full((8, 8), -2.0), S["S88"])) == pytest.approx(0, abs=1e-9)
    assert bz.variance(comp(bz, np.zeros((8, 8)), S["S88"])) == 0.0
    assert bz.l2_norm(comp(bz, np.ones((8, 8)), S["S88"])) == pytest.approx(8.0, rel=1e-6)
    a = comp(bz, rng.uniform(-1, 1, (16, 16)), S["S44"])
    assert bz.cosine_similarity(a, a) == pytest.approx(1.0, abs=1e-9)
    assert bz.cosine_similarity(a, bz.negate(a)) == pytest.approx(-1.0, abs=1e-9)
    assert bz.ssim(a, a) == pytest.approx(1.0, abs=1e-9)
    out = bz.decompress(bz.add_scalar(comp(bz, np.full((8, 8), 1.5), S["S88"]), 2.25))
    assert np.allclose(out.numpy(), 3.75, rtol=0, atol=1e-6)
    big = bz.add_scalar(comp(bz, rng.uniform(0, 1, (16, 16)), S["S44"]), 1000.0)
    assert int(big.indices.max()) <= 32767 and int(big.indices.min()) >= -32767


@pytest.mark.parametrize("block,ik", [((8, 8, 8), "i64"), ((32, 32), "i32"), ((64, 64), "i16")])
def test_add_large_blocks(bz, rng, block, ik):
    """Blocks too large for the register-held add layouts."""
    shape = tuple(2 * b + 1 for b in block)
    x, y = rng.normal(size=shape), rng.normal(size=shape)
    s = bz.CodecSettings(block, bz.FloatKind.F64, bz.IndexKind(ik))
    os_ = o.Settings(block, "f64", ik)
    a, b = comp(bz, x, s), comp(bz, y, s)

    def ref(c):
        return o.Compressed(shape, os_, c.maxima_f64().cpu().numpy(), c.indices.cpu().numpy())

    for got, want in ((bz.add(a, b), o.add(ref(a), ref(b))),
                      (bz.subtract(a, b), o.subtract(ref(a), ref(b))),
                      (bz.add_scalar(a, 0.75), o.add_scalar(ref(a), 0.75))):
        assert np.array_equal(got.maxima_f64().cpu().numpy(), want.maxima)
        assert np.array_equal(got.indices.cpu().numpy(), want.indices)
    d = bz.subtract_l2(a, b)
    assert math.isclose(d, o.l2_norm(o.subtract(ref(a), ref(b))), rel_tol=1e-12)


def test_huge_maxima_reductions(bz):
    """Maxima near 1e300 with sparse AC coefficients: the reference squares
    F*N per element (inf where F != 0, 0 where F == 0); never NaN."""
    x = np.zeros((16, 16))
    x[0:4, 0:4] = 1e300           # one constant block: only the DC coefficient is nonzero
    x[4:8, 0:4] = np.linspace(-1, 1, 16).reshape(4, 4)
    s = bz.CodecSettings((4, 4), bz.FloatKind.F64, bz.IndexKind.I16)
    a = comp(bz, x, s)
    z = comp(bz, np.zeros((16, 16)), s)
    l2 = bz.l2_norm(a)
    assert l2 == math.inf
    assert bz.dot(a, z) == 0.0
    y = np.zeros((16, 16))
    y[0:4, 0:4] = 1e-300
    t = comp(bz, y, s)
    assert bz.l2_norm(t) >= 0.0 and not math.isnan(bz.l2_norm(t))


def test_c_abi_rejects_mismatched_layouts(bz, S, rng):
    from paper_2406_11209_b200 import _native

    a = comp(bz, rng.uniform(size=(16, 16)), S["S44"])
    c = comp(bz, rng.uniform(size=(8, 8)), S["S44"])
    La, Lc = a.layout(), c.layout()
    rec = torch.empty(16, dtype=torch.float64, device="cuda")
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    out_m, out_i = torch.empty_like(a.maxima), torch.empty_like(a.indices)
    lib = _native.load_library()
    rc = lib.bz_add(ctypes.byref(La), ctypes.byref(Lc), a.maxima.data_ptr(), a.indices.data_ptr(),
                    c.maxima.data_ptr(), c.indices.data_ptr(), 0, out_m.data_ptr(),
                    out_i.data_ptr(), None, _native.stream_handle())
    assert rc != 0 and b"block counts differ" in lib.bz_last_error()
    rc = lib.bz_moments(ctypes.byref(La), ctypes.byref(Lc), a.maxima.data_ptr(),
                        a.indices.data_ptr(), c.maxima.data_ptr(), c.indices.data_ptr(), 1, 0,
                        rec.data_ptr(), ws.data_ptr(), ws.numel(), _native.stream_handle())
    assert rc != 0
    nf = comp(bz, rng.uniform(size=(16, 16)), _no_first(bz, (4, 4)))
    full15 = bz.CodecSettings((4, 4), bz.FloatKind.F64,
                              mask=bz.PruningMask.first_k((4, 4), 15))
    f15 = comp(bz, rng.uniform(size=(16, 16)), full15)
    rc = lib.bz_moments(ctypes.byref(nf.layout()), ctypes.byref(f15.layout()),
                        nf.maxima.data_ptr(), nf.indices.data_ptr(), f15.maxima.data_ptr(),
                        f15.indices.data_ptr(), 1, 0, rec.data_ptr(), ws.data_ptr(), ws.numel(),
                        _native.stream_handle())
    assert rc != 0 and b"masks differ" in lib.bz_last_error()
    # the valid call still works after the rejected ones
    assert math.isclose(bz.dot(a, a), bz.l2_norm(a) ** 2, rel_tol=1e-12)


def test_concurrent_reductions_from_threads(bz):
    """Four threads reducing on one stream get the serial results
    (the reference's ops are pure functions)."""
    rng = np.random.default_rng(7)
    s = bz.CodecSettings((8, 8, 8), bz.FloatKind.F32, bz.IndexKind.I8)
    arrs = [bz.compress(bz.DenseArray.of(rng.normal(size=(64, 64, 64)), bz.FloatKind.F32), s)
            for _ in range(4)]
    def ops3(i):  # subtract_l2's last CTA writes into the calling thread's pinned record
        return (bz.dot(arrs[i], arrs[(i + 1) % 4]), bz.l2_norm(arrs[i]),
                bz.subtract_l2(arrs[i], arrs[(i + 1) % 4]))

    serial = [ops3(i) for i in range(4)]
    errors, results = [], {}

    def worker(i):
        try:
            got = []
            for _ in range(50):
                got.append(ops3(i))
            results[i] = got
        except Exception as e:  # pragma: no cover
            errors.append(e)

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors
    for i in range(4):
        assert all(g == serial[i] for g in results[i]), i


def test_reduction_workspace_survives_a_failed_launch(bz, S, rng):
    from paper_2406_11209_b200 import _native, ops

    a = comp(bz, rng.uniform(size=(16, 16)), S["S44"])
    want = bz.l2_norm(a)
    ws = ops._reduce_workspace(a.device, a.layout())
    ws[:4].fill_(7)  # a ticket left half-counted (as after an aborted launch) ...
    bad = bz.CompressedArray((16, 16), S["S44"], a.maxima, a.indices, _trusted=True)
    object.__setattr__(bad, "_lay", _native.Layout())  # ... and a call the library rejects
    with pytest.raises(_native.NativeError):
        ops.moments_record(bad)
    assert bz.l2_norm(a) == want  # the failure path re-zeroed the workspace


def test_host_record_is_device_addressable(bz, S, rng):
    """The reduction's last CTA writes the record straight into pinned host
    memory (UVA); the value equals the device-record path."""
    from paper_2406_11209_b200 import ops

    a = comp(bz, rng.uniform(size=(64, 64)), S["S44"])
    h = ops.moments_record(a, dc_only=2, out=ops._host_record())
    torch.cuda.synchronize()
    d = ops.record_to_host(ops.moments_record(a, dc_only=2))
    assert np.array_equal(h.numpy()[:9], d[:9])
