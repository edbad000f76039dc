"""Parity at the BASELINE.json sizes (VERDICT r01 "What's missing" #3).

The GPU runs each configuration at its full size (or a large block-row slab
of it); the oracle checks the result chunk by chunk along axis 0 (blocks are
independent), so memory stays bounded:

* C2 8192^2 f64 4x4 I16 at full size: maxima bit-exact, indices bit-exact
  except at rounding ties (counted), decompression 1e-13, l2 1e-9;
* C3/C4 (128,1024,1024) slab f32 8^3 I8: compress bit-exact (tie-aware);
* C4 covariance / cosine / SSIM / mean / variance on two FULL 1024^3
  GPU-compressed fields (2,097,152 blocks) vs a chunked f64 restatement of
  the reference's reductions (ops.py:226-348, chunked like ops.py:131-163),
  rel 1e-9;
* C5 (32,256,256,64) slab f32 4^4 I8 with the low-pass mask (K=66).
"""

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


def _fill(bz, shape, kind, seed, offset=0):
    from paper_2406_11209_b200 import _native

    t = torch.empty(shape, dtype=kind.torch_dtype, device="cuda")
    _native.call("bz_fill_random", t.data_ptr(), kind.code, t.numel(), offset, seed, 0,
                 _native.stream_handle())
    return bz.DenseArray.wrap(t, kind)


def _settings(bz, block, fk, ik, mask_bits=None):
    mask = None if mask_bits is None else bz.PruningMask(tuple(block), mask_bits)
    return bz.CodecSettings(tuple(block), bz.FloatKind(fk), bz.IndexKind(ik),
                            bz.TransformFamily.DCT, mask)


def _chunked_codec_parity(bz, x, s, block, fk, ik, mask_bits, chunk_rows, check_decompress):
    """GPU compress of the whole array vs the oracle on chunks of block rows.
    Returns (indices, index mismatches, mismatches at ties, worst decompress err)."""
    ca = bz.compress(x, s)
    os_ = o.Settings(block, fk, ik, "dct", mask_bits)
    n0 = x.shape[0]
    b0 = block[0]
    total = mism = at_ties = 0
    worst = 0.0
    dec = bz.decompress(ca).values if check_decompress else None
    for r0 in range(0, n0, chunk_rows):
        r1 = min(n0, r0 + chunk_rows)
        xs = x.values[r0:r1].double().cpu().numpy()
        ref = o.compress(xs, os_)
        g0, g1 = r0 // b0, -(-r1 // b0)
        got_m = ca.maxima_f64()[g0:g1].cpu().numpy()
        got_i = ca.indices[g0:g1].cpu().numpy()
        assert np.array_equal(got_m.view(np.int64), ref.maxima.view(np.int64)), \
            f"maxima differ in rows {r0}:{r1}"
        diff = got_i != ref.indices
        if diff.any():
            ties = o.prune_and_flatten(o.tie_mask(o.coefficients(xs, os_), ref.maxima,
                                                  len(block), ik), os_.mask_bits)
            assert not (diff & ~ties).any(), int((diff & ~ties).sum())
            at_ties += int(diff.sum())
        mism += int(diff.sum())
        total += diff.size
        if check_decompress:
            want = o.decompress(ref)
            got = dec[r0:r1].cpu().numpy()
            span = max(float(np.max(np.abs(want))), 1e-300)
            worst = max(worst, float(np.max(np.abs(got - want))) / span)
    return ca, total, mism, at_ties, worst


def test_c2_full_size_vs_oracle(bz):
    s = _settings(bz, (4, 4), "f64", "i16")
    x = _fill(bz, (8192, 8192), bz.FloatKind.F64, 21)
    ca, total, mism, ties, worst = _chunked_codec_parity(bz, x, s, (4, 4), "f64", "i16", None,
                                                         1024, True)
    print(f"C2 full: {total} indices, {mism} mismatches ({ties} at ties), "
          f"decompress rel err {worst:.2e}")
    assert total == 2048 * 2048 * 16
    assert worst <= 1e-13
    # l2 of the full array vs the oracle's l2 (chunked sums of P^2, ops.py:291-297)
    acc = 0.0
    for g0 in range(0, 2048, 256):
        m = ca.maxima_f64()[g0:g0 + 256].cpu().numpy()
        i = ca.indices[g0:g0 + 256].cpu().numpy().astype(np.float64)
        p = i * m[..., None]
        acc += float(np.dot(p.ravel(), p.ravel()))
    want = math.sqrt(acc) / 32767.0
    assert math.isclose(bz.l2_norm(ca), want, rel_tol=1e-9)


def test_c3_slab_compress_bit_exact(bz):
    s = _settings(bz, (8, 8, 8), "f32", "i8")
    x = _fill(bz, (128, 1024, 1024), bz.FloatKind.F32, 31)
    _, total, mism, ties, _ = _chunked_codec_parity(bz, x, s, (8, 8, 8), "f32", "i8", None, 16,
                                                    False)
    print(f"C3 slab: {total} indices, {mism} mismatches ({ties} at ties)")
    assert total == 128 * 1024 * 1024


def test_c5_slab_lowpass_vs_oracle(bz):
    bits = np.indices((4, 4, 4, 4)).sum(axis=0) <= 4
    s = _settings(bz, (4, 4, 4, 4), "f32", "i8", bits)
    x = _fill(bz, (32, 256, 256, 64), bz.FloatKind.F32, 41)
    _, total, mism, ties, worst = _chunked_codec_parity(bz, x, s, (4, 4, 4, 4), "f32", "i8",
                                                        bits, 4, True)
    print(f"C5 slab: {total} indices, {mism} mismatches ({ties} at ties), "
          f"decompress rel err {worst:.2e}")
    assert total == (32 * 256 * 256 * 64 // 256) * 66
    assert worst <= 1e-13


def _chunked_reductions(a, b, chunk=65536):
    """The reference's dot / l2 / mean / covariance / SSIM terms (ops.py:226-348)
    from the compressed data, in f64, over chunks of blocks."""
    ma = a.maxima_f64().reshape(-1)
    mb = b.maxima_f64().reshape(-1)
    k = a.indices.shape[-1]
    ia = a.indices.reshape(-1, k)
    ib = b.indices.reshape(-1, k)
    nb = ia.shape[0]
    # pass 1: sums of first coefficients (F0*N), i.e. block means * r * sqrt(bs)
    fa = fb = 0.0
    for c0 in range(0, nb, chunk):
        fa += float((ia[c0:c0 + chunk, 0].double() * ma[c0:c0 + chunk]).sum().item())
        fb += float((ib[c0:c0 + chunk, 0].double() * mb[c0:c0 + chunk]).sum().item())
    mean_a, mean_b = fa / nb, fb / nb
    dab = daa = dbb = cab = caa = cbb = 0.0
    for c0 in range(0, nb, chunk):
        pa = ia[c0:c0 + chunk].double().cpu().numpy() * ma[c0:c0 + chunk].cpu().numpy()[:, None]
        pb = ib[c0:c0 + chunk].double().cpu().numpy() * mb[c0:c0 + chunk].cpu().numpy()[:, None]
        dab += float(np.dot(pa.ravel(), pb.ravel()))
        daa += float(np.dot(pa.ravel(), pa.ravel()))
        dbb += float(np.dot(pb.ravel(), pb.ravel()))
        pa[:, 0] -= mean_a
        pb[:, 0] -= mean_b
        cab += float(np.dot(pa.ravel(), pb.ravel()))
        caa += float(np.dot(pa.ravel(), pa.ravel()))
        cbb += float(np.dot(pb.ravel(), pb.ravel()))
    return dict(n=nb, mean_a=mean_a, mean_b=mean_b, dab=dab, daa=daa, dbb=dbb, cab=cab,
                caa=caa, cbb=cbb)


def test_c4_full_size_reductions_vs_chunked_oracle(bz):
    s = _settings(bz, (8, 8, 8), "f32", "i8")
    x = _fill(bz, (1024, 1024, 1024), bz.FloatKind.F32, 51)
    a = bz.compress(x, s)
    del x
    y = _fill(bz, (1024, 1024, 1024), bz.FloatKind.F32, 52)
    # correlated second field: y' = x/2 + y/2 in the compressed domain
    b = bz.mul_scalar(bz.add(a, bz.compress(y, s)), 0.5)
    del y
    torch.cuda.synchronize()
    R = _chunked_reductions(a, b)
    r, bs, nb = 127.0, 512, R["n"]
    assert nb == 2097152
    sq = math.sqrt(bs)
    want = {
        "dot": R["dab"] / (r * r),
        "l2": math.sqrt(R["daa"]) / r,
        "mean": (R["mean_a"] / r) / sq,
        "mean_pc": sq * (R["mean_a"] / r * nb) / 1024 ** 3,
        "variance": R["caa"] / (r * r) / (nb * bs),
        "covariance": R["cab"] / (r * r) / (nb * bs),
        "cosine": R["dab"] / math.sqrt(R["daa"] * R["dbb"]),
    }
    mu_a, mu_b = want["mean"], (R["mean_b"] / r) / sq
    va, vb = want["variance"], R["cbb"] / (r * r) / (nb * bs)
    cov = want["covariance"]
    sl, sc = 1e-4, 9e-4
    lum = (2 * mu_a * mu_b + sl) / (mu_a ** 2 + mu_b ** 2 + sl)
    con = (2 * math.sqrt(va * vb) + sc) / (va + vb + sc)
    st = (cov + sc / 2) / (math.sqrt(va) * math.sqrt(vb) + sc / 2)
    want["ssim"] = lum * con * st
    got = {
        "dot": bz.dot(a, b), "l2": bz.l2_norm(a), "mean": bz.mean(a),
        "mean_pc": bz.mean(a, padding_corrected=True), "variance": bz.variance(a),
        "covariance": bz.covariance(a, b), "cosine": bz.cosine_similarity(a, b),
        "ssim": bz.ssim(a, b),
    }
    for k in want:
        assert math.isclose(got[k], want[k], rel_tol=1e-9, abs_tol=1e-15), (k, got[k], want[k])
    # the fused covariance really sees a correlated pair
    assert 0.5 < got["cosine"] < 0.9


def test_c3_slab_add_chain_bit_exact(bz):
    """add / subtract / add_scalar / mul_scalar of two GPU-compressed C3 slabs
    vs the oracle on the same compressed data, chunk by chunk (ops.py:178-223)."""
    s = _settings(bz, (8, 8, 8), "f32", "i8")
    a = bz.compress(_fill(bz, (64, 1024, 1024), bz.FloatKind.F32, 61), s)
    b = bz.compress(_fill(bz, (64, 1024, 1024), bz.FloatKind.F32, 62), s)
    os_ = o.Settings((8, 8, 8), "f32", "i8")
    results = [("add", bz.add(a, b)), ("sub", bz.subtract(a, b)),
               ("adds", bz.add_scalar(a, 0.375)), ("chain", bz.mul_scalar(bz.add(a, b), 0.5))]
    for g0 in range(0, 8, 2):
        sl = slice(g0, g0 + 2)
        shp = (16, 1024, 1024)
        ra = o.Compressed(shp, os_, a.maxima_f64()[sl].cpu().numpy(), a.indices[sl].cpu().numpy())
        rb = o.Compressed(shp, os_, b.maxima_f64()[sl].cpu().numpy(), b.indices[sl].cpu().numpy())
        want = {"add": o.add(ra, rb), "sub": o.subtract(ra, rb), "adds": o.add_scalar(ra, 0.375)}
        want["chain"] = o.mul_scalar(want["add"], 0.5)
        for name, got in results:
            w = want[name]
            assert np.array_equal(got.maxima_f64()[sl].cpu().numpy(), w.maxima), (name, g0)
            assert np.array_equal(got.indices[sl].cpu().numpy(), w.indices), (name, g0)
