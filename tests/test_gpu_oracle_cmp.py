"""compare_against_oracle (metrics.py:224-323) on the GPU vs the reference's own
records (tests/golden/make_golden_oracle.py).  The compressed-space value must
match the reference's within the reduction tolerance (1e-9 relative), the
conventional value likewise, and the deviations agree to the precision they
carry (both routes are float64 sums of ~1e-16-relative differences); the
rebinning bound is exact because the maxima are bit-exact."""

import json
import math
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TABLE = json.load(open(os.path.join(HERE, "oracle_cmp.json")))
ARR = np.load(os.path.join(HERE, "oracle_cmp.npz"))
SCALARS = {"add_scalar": 0.75, "mul_scalar": -2.5}


@pytest.fixture(scope="module")
def bz():
    import paper_2406_11209_b200 as m

    assert torch.cuda.is_available()
    return m


@pytest.mark.parametrize("case", TABLE, ids=lambda c: c["name"])
def test_compare_against_oracle_matches_reference(bz, case):
    from paper_2406_11209_b200 import metrics

    fk = bz.FloatKind(case["float_kind"])
    block = tuple(case["block"])
    mask = None
    if case["lowpass"] is not None:
        mask = bz.PruningMask(block, np.indices(block).sum(axis=0) <= case["lowpass"])
    s = bz.CodecSettings(block, fk, bz.IndexKind(case["index_kind"]), mask=mask)
    xs = [bz.DenseArray(tuple(case["shape"]), fk, ARR[f"{case['name']}/x{j}"]) for j in range(2)]
    comps = []
    for op, want in case["records"].items():
        arity = metrics.ORACLE_OPERATIONS[op][0]
        got = metrics.compare_against_oracle(op, xs[:arity], s, x=SCALARS.get(op, 0.0))
        comps.append(got)
        assert got.name == want["name"] and got.result_type == want["result_type"]
        assert got.note == want["note"]
        if want["result_type"] == "scalar":
            scale = max(abs(want["oracle"]), 1e-300)
            tol = 1e-9 if op not in ("ssim", "cosine_similarity") else 0.0
            for k in ("compressed", "oracle"):
                assert math.isclose(got.__dict__[k], want[k], rel_tol=1e-9, abs_tol=tol or 1e-15), \
                    (op, k, got.__dict__[k], want[k])
            assert abs(got.absolute_deviation - want["absolute_deviation"]) <= 1e-12 * scale, op
        else:
            assert got.compressed is None and got.oracle is None
            if want["bound"] is None:
                assert got.bound is None
            else:
                assert got.bound == want["bound"], (op, got.bound, want["bound"])
            # negate / mul_scalar are exact; add / add_scalar deviations are rebinning errors
            assert abs(got.absolute_deviation - want["absolute_deviation"]) <= \
                1e-12 * max(1.0, abs(want["absolute_deviation"]) / max(want["relative_deviation"], 1e-300)), op
    assert metrics.render_table(comps).count("\n") == len(comps)
