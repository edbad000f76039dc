"""Host side of the .bzc streams (no GPU): the header parser against the
reference's golden streams (tests/golden/make_golden_ext.py), the layout
arithmetic, and the reference's malformed-stream errors."""

import json
import math
import os

import numpy as np
import pytest

from paper_2406_11209_b200 import errors
from paper_2406_11209_b200.format import _fields, parse_header
from paper_2406_11209_b200.ops import WassersteinParams

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ARR = dict(np.load(os.path.join(HERE, "ext.npz")))
TABLE = json.load(open(os.path.join(HERE, "ext.json")))
CASES = [c for c in TABLE if f"{c['name']}/stream0" in ARR]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_header_parse_and_layout(case):
    stream = ARR[f"{case['name']}/stream0"]
    shape, settings, P = parse_header(stream, stream.size)
    assert shape == tuple(case["shape"])
    assert settings.block_shape == tuple(case["block"])
    assert settings.float_kind.value == case["float_kind"]
    assert settings.index_kind.value == case["index_kind"]
    blocks = math.prod(settings.grid_for(shape))
    fields = _fields(settings, len(shape), blocks)
    assert fields[7] == ("maxima", P, settings.float_kind.bits * blocks)
    total = fields[-1][1] + fields[-1][2]
    assert total // 8 == stream.size  # the reference's stream length


def test_malformed_headers():
    stream = ARR[f"{CASES[0]['name']}/stream0"]
    with pytest.raises(errors.TruncatedStream):
        parse_header(np.zeros(0, np.uint8), 0)
    with pytest.raises(errors.TruncatedStream):
        parse_header(stream[:-8], stream.size - 8)
    bad = stream.copy()
    bad[0] = (bad[0] & 0x0F) | 0x70
    with pytest.raises(errors.InvalidTypeCode):
        parse_header(bad, bad.size)
    with pytest.raises(errors.ZeroExtent):
        parse_header(np.zeros(16, np.uint8), 16)


def test_wasserstein_params_validation():
    with pytest.raises(ValueError):
        WassersteinParams(order=0.5)
    with pytest.raises(ValueError):
        WassersteinParams(normalization_tolerance=-1.0)
    assert WassersteinParams().order == 1.0
