"""Host-side logic of the drop-in API that needs no GPU: settings and mask
validation with the reference's exception types, kinds metadata, and the
partial-record algebra used by every reduction (single GPU and sharded)."""

import math

import numpy as np
import pytest

import paper_2406_11209_b200 as bz
from paper_2406_11209_b200 import errors
from paper_2406_11209_b200.ops import Record, merge_records


def test_kinds_metadata_matches_reference():
    assert [k.bits for k in bz.FloatKind] == [16, 16, 32, 64]
    assert bz.IndexKind.I8.radius == 127 and bz.IndexKind.I16.radius == 32767
    assert bz.IndexKind.I64.clamp_bound == 2.0 ** 63 - 1024
    assert bz.FloatKind.F16.max_finite == 65504.0
    assert bz.FloatKind.from_code(2) is bz.FloatKind.F32
    assert bz.IndexKind.parse(" I16 ") is bz.IndexKind.I16


def test_settings_validation():
    with pytest.raises(errors.NonPowerOfTwoBlock):
        bz.CodecSettings((3, 4))
    with pytest.raises(errors.DimensionMismatch):
        bz.CodecSettings((4, 4), mask=bz.PruningMask.full((4,)))
    s = bz.CodecSettings((4, 4))
    assert s.float_kind is bz.FloatKind.F32 and s.index_kind is bz.IndexKind.I16
    assert s.block_mean_scale == 4.0
    assert s.grid_for((5, 9)) == (2, 3)
    with pytest.raises(errors.DimensionMismatch):
        s.grid_for((5,))
    with pytest.raises(errors.DegenerateShape):
        s.grid_for((0, 4))
    assert s == bz.CodecSettings((4, 4)) and hash(s) == hash(bz.CodecSettings((4, 4)))


def test_mask_api():
    bits = np.ones((8, 8), dtype=bool)
    bits[2:, 2:] = False
    m = bz.PruningMask.from_bits((8, 8), bits)
    assert m.kept_count == 28 and m.keeps_first
    assert bz.PruningMask.first_k((4, 4), 6).kept_count == 6
    with pytest.raises(errors.LengthMismatch):
        bz.PruningMask.from_bits((4, 4), np.ones(15, dtype=bool))
    with pytest.raises(ValueError):
        bz.PruningMask.first_k((4,), 5)
    assert list(bz.PruningMask.first_k((4,), 2).flat_kept) == [0, 1]


def test_transform_matrices_bit_identical_to_oracle():
    import bzc_oracle as o

    for size in (1, 2, 4, 8, 16, 32):
        for fam in bz.TransformFamily:
            got = bz.make_transform(size, fam).entries
            assert np.array_equal(got.view(np.uint64), o.matrix(size, fam.value).view(np.uint64))
    with pytest.raises(errors.NonPowerOfTwoBlock):
        bz.make_transform(6, bz.TransformFamily.DCT)


def _record_of(dca, dcb, sab, saa, sbb):
    n = len(dca)
    ma, mb = float(np.mean(dca)), float(np.mean(dcb))
    return Record(n, ma, mb, float(np.sum((dca - ma) * (dcb - mb))),
                  float(np.sum((dca - ma) ** 2)), float(np.sum((dcb - mb) ** 2)), sab, saa, sbb)


def test_chan_merge_matches_direct():
    rng = np.random.default_rng(0)
    dca = rng.normal(1e3, 1.0, 1000)
    dcb = 0.5 * dca + rng.normal(0, 1, 1000)
    whole = _record_of(dca, dcb, 1.0, 2.0, 3.0)
    parts = [_record_of(dca[i:j], dcb[i:j], 0.25, 0.5, 0.75)
             for i, j in ((0, 100), (100, 400), (400, 1000))]
    parts.append(Record(0, 0, 0, 0, 0, 0, 0, 0, 0))
    merged = merge_records(parts)
    assert merged.n == 1000
    for f in ("mean_a", "mean_b", "m_ab", "m_aa", "m_bb"):
        assert math.isclose(getattr(merged, f), getattr(whole, f), rel_tol=1e-10), f
    assert merged.s_ab == 0.75 and merged.s_bb == 2.25
