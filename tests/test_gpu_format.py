""".bzc streams: GPU-packed streams equal the reference's
serialize() byte for byte, deserialize() inverts them, malformed streams raise
the reference's exceptions (pkg/tests/test_format.py cases).  Golden streams:
tests/golden/make_golden_ext.py (the real reference)."""

import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ARR = dict(np.load(os.path.join(HERE, "ext.npz")))
TABLE = json.load(open(os.path.join(HERE, "ext.json")))
STREAM_CASES = [c for c in TABLE if f"{c['name']}/stream0" in ARR]


@pytest.fixture(scope="module")
def bz():
    import paper_2406_11209_b200 as m

    assert torch.cuda.is_available()
    return m


_BITS_DTYPE = {"bf16": (np.int16, torch.bfloat16), "f16": (np.int16, torch.float16),
               "f32": (np.int32, torch.float32), "f64": (np.int64, torch.float64)}


def compressed(bz, case, j):
    """The reference's compressed array j of a case, on the GPU."""
    name = case["name"]
    block = tuple(case["block"])
    mask = ARR.get(f"{name}/mask")
    pm = None if mask is None else bz.PruningMask(block, mask)
    s = bz.CodecSettings(block, bz.FloatKind(case["float_kind"]), bz.IndexKind(case["index_kind"]),
                         mask=pm)
    npd, td = _BITS_DTYPE[case["float_kind"]]
    maxima = torch.from_numpy(ARR[f"{name}/max{j}"].astype(npd, copy=True)).view(td).cuda()
    idx = torch.from_numpy(ARR[f"{name}/idx{j}"].copy()).cuda()
    return bz.CompressedArray(tuple(case["shape"]), s, maxima, idx)


@pytest.mark.parametrize("case", STREAM_CASES, ids=[c["name"] for c in STREAM_CASES])
def test_serialize_matches_reference(bz, case):
    for j in range(3):
        a = compressed(bz, case, j)
        want = ARR[f"{case['name']}/stream{j}"].tobytes()
        got = bz.serialize(a)
        assert got == want
        layout = bz.bitstream_layout(a)
        assert layout.total_bytes == len(want)
        assert [f[0] for f in layout.fields] == ["float_kind", "index_kind", "transform",
                                                 "original_shape", "shape_marker", "block_shape",
                                                 "mask", "maxima", "indices", "padding"]


@pytest.mark.parametrize("case", STREAM_CASES, ids=[c["name"] for c in STREAM_CASES])
def test_deserialize_round_trip(bz, case):
    for j in range(3):
        a = compressed(bz, case, j)
        stream = ARR[f"{case['name']}/stream{j}"].tobytes()
        back = bz.deserialize(stream)
        assert back == a  # bit-exact maxima (NaN payloads included) and indices
        dev = bz.serialize_to_device(a)
        assert dev.is_cuda
        assert bz.deserialize(dev) == a
        # trailing bytes are ignored (format.py:166)
        assert bz.deserialize(stream + b"\x00\xff\x17") == a


def test_round_trip_c1_size(bz):
    from paper_2406_11209_b200 import _native

    x = torch.empty((256, 256, 256), dtype=torch.float32, device="cuda")
    _native.call("bz_fill_random", x.data_ptr(), 2, x.numel(), 0, 5, 0, _native.stream_handle())
    s = bz.CodecSettings((8, 8, 8), bz.FloatKind.F32, bz.IndexKind.I8)
    a = bz.compress(bz.DenseArray.wrap(x, bz.FloatKind.F32), s)
    stream = bz.serialize_to_device(a)
    assert stream.numel() == bz.bitstream_layout(a).total_bytes
    assert bz.deserialize(stream) == a


def test_malformed_streams(bz):
    from paper_2406_11209_b200 import errors

    case = STREAM_CASES[0]
    a = compressed(bz, case, 0)
    stream = bz.serialize(a)
    with pytest.raises(errors.TruncatedStream):
        bz.deserialize(b"")
    with pytest.raises(errors.TruncatedStream):
        bz.deserialize(stream[:-40])
    header_bytes = bz.bitstream_layout(a).fields[7][1] // 8
    with pytest.raises(errors.TruncatedStream):
        bz.deserialize(stream[:header_bytes])
    bad = bytearray(stream)
    bad[0] = (bad[0] & 0x0F) | (0x5 << 4)  # transform code bits 4..11 -> 5 (invalid)
    with pytest.raises(errors.InvalidTypeCode):
        bz.deserialize(bytes(bad))
    # zero first extent: shape marker straight after the codes
    zero = bytearray(16)
    zero[0] = 0x0  # F16? codes 0/0, DCT; then a zero word -> empty shape
    with pytest.raises(errors.ZeroExtent):
        bz.deserialize(bytes(zero))
