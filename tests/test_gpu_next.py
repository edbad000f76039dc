"""SURVEY §8f rows 1-2 on the GPU against the real reference (goldens from
tests/golden/make_golden_ext.py): block_means (bit-exact), approx_wasserstein
(orders 1, 2, 3.5; with and without the softmax), and the time-series l2
workflow (cli.py:225-259) through the fused subtract+l2 kernel."""

import json
import math
import os

import numpy as np
import pytest
import torch

from test_gpu_format import ARR, TABLE, compressed

pytestmark = pytest.mark.gpu

MEAN_CASES = [c for c in TABLE if "wasserstein" in c]


@pytest.fixture(scope="module")
def bz():
    import paper_2406_11209_b200 as m

    assert torch.cuda.is_available()
    return m


@pytest.mark.parametrize("case", [c for c in MEAN_CASES if f"{c['name']}/means0" in ARR],
                         ids=lambda c: c["name"])
def test_block_means_bit_exact(bz, case):
    got = bz.block_means(compressed(bz, case, 0)).cpu().numpy()
    want = ARR[f"{case['name']}/means0"]
    assert np.array_equal(got, want, equal_nan=True)


@pytest.mark.parametrize("case", MEAN_CASES, ids=lambda c: c["name"])
def test_approx_wasserstein_matches_reference(bz, case):
    a, b = compressed(bz, case, 0), compressed(bz, case, 1)
    for order, want in case["wasserstein"].items():
        got = bz.approx_wasserstein(a, b, bz.WassersteinParams(order=float(order)))
        if math.isnan(want):
            assert math.isnan(got)
        else:
            assert math.isclose(got, want, rel_tol=1e-9, abs_tol=1e-15), (order, got, want)


def test_wasserstein_properties(bz):
    """Symmetry, identity, and a large sort (2^20 + 7 blocks, many ties)."""
    rng = np.random.default_rng(3)
    s = bz.CodecSettings((4, 4), bz.FloatKind.F32, bz.IndexKind.I8)
    shape = (4 * 1031, 4 * 1017 + 28)
    x = rng.normal(size=shape)
    y = np.round(rng.normal(size=shape), 1)
    a = bz.compress(bz.DenseArray.of(x, bz.FloatKind.F32), s)
    b = bz.compress(bz.DenseArray.of(y, bz.FloatKind.F32), s)
    assert bz.approx_wasserstein(a, a) == 0.0
    w_ab = bz.approx_wasserstein(a, b, bz.WassersteinParams(order=2.0))
    w_ba = bz.approx_wasserstein(b, a, bz.WassersteinParams(order=2.0))
    assert w_ab == w_ba
    # against numpy on the GPU's own block means (softmax, sort, p-norm)
    pa, pb = bz.block_means(a).cpu().numpy(), bz.block_means(b).cpu().numpy()

    def sm(v):
        z = np.exp(v - v.max())
        return z / z.sum()

    pa, pb = sm(pa), sm(pb)
    want = float(np.sqrt(np.sum(np.abs(np.sort(pa) - np.sort(pb)) ** 2) / pa.size))
    assert math.isclose(w_ab, want, rel_tol=1e-9)


@pytest.mark.parametrize("case", [c for c in MEAN_CASES if "timeseries_l2" in c],
                         ids=lambda c: c["name"])
def test_timeseries_l2_matches_reference(bz, case):
    snaps = [compressed(bz, case, j) for j in range(3)]
    got = bz.timeseries_distances(snaps, "l2")
    for g, w in zip(got, case["timeseries_l2"]):
        if math.isnan(w):
            assert math.isnan(g)
        else:
            assert math.isclose(g, w, rel_tol=1e-9, abs_tol=1e-12), (g, w)
    # fused pass == materialised difference, and wasserstein measure wiring
    for i in range(2):
        assert math.isclose(bz.subtract_l2(snaps[i + 1], snaps[i]),
                            bz.l2_norm(bz.subtract(snaps[i + 1], snaps[i])), rel_tol=1e-12) or \
            math.isnan(got[i])
    ws = bz.timeseries_distances(snaps, "wasserstein", 2.0)
    assert len(ws) == 2


def test_fused_subtract_l2_c3_slab(bz):
    """C3 settings on a 256 x 1024 x 1024 slab: fused == compose."""
    from paper_2406_11209_b200 import _native

    s = bz.CodecSettings((8, 8, 8), bz.FloatKind.F32, bz.IndexKind.I8)
    xs = []
    for seed in (31, 32):
        t = torch.empty((256, 1024, 1024), dtype=torch.float32, device="cuda")
        _native.call("bz_fill_random", t.data_ptr(), 2, t.numel(), 0, seed, 0, _native.stream_handle())
        xs.append(bz.compress(bz.DenseArray.wrap(t, bz.FloatKind.F32), s))
    fused = bz.subtract_l2(xs[1], xs[0])
    comp = bz.l2_norm(bz.subtract(xs[1], xs[0]))
    assert math.isclose(fused, comp, rel_tol=1e-12)


METRIC_CASES = [c for c in TABLE if c.get("observed_linf") is not None]


@pytest.mark.parametrize("case", METRIC_CASES, ids=lambda c: c["name"])
def test_error_report_matches_reference(bz, case):
    """per-block predictors and round-trip errors on the GPU
    vs bzc.metrics.measure_roundtrip; ratios vs bzc.metrics."""
    from paper_2406_11209_b200 import metrics

    name = case["name"]
    block = tuple(case["block"])
    s = bz.CodecSettings(block, bz.FloatKind(case["float_kind"]), bz.IndexKind(case["index_kind"]),
                         mask=bz.PruningMask(block, ARR[f"{name}/mask"]))
    x = ARR[f"{name}/x0"]
    rep = metrics.measure_roundtrip(bz.DenseArray.of(x, bz.FloatKind(case["float_kind"])), s)
    assert np.array_equal(rep.per_block_bin_bound.cpu().numpy(), ARR[f"{name}/bin_bound"])
    assert np.array_equal(rep.per_block_loose_linf.cpu().numpy(), ARR[f"{name}/loose_linf"])
    np.testing.assert_allclose(rep.per_block_l2_coeff_error.cpu().numpy(), ARR[f"{name}/l2_coeff"],
                               rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(rep.per_block_observed_l2.cpu().numpy(), ARR[f"{name}/obs_l2_blocks"],
                               rtol=1e-9, atol=1e-300)
    assert math.isclose(rep.observed_linf, case["observed_linf"], rel_tol=1e-9, abs_tol=1e-300)
    assert math.isclose(rep.observed_l2, case["observed_l2"], rel_tol=1e-9, abs_tol=1e-300)
    closed, measured, nbytes = case["ratio"]
    shape = tuple(case["shape"])
    assert metrics.compression_ratio(32, s, shape) == closed
    c0 = compressed(bz, case, 0)
    assert len(bz.serialize(c0)) == nbytes
    assert metrics.measured_ratio(32, shape, nbytes) == measured
