"""Load the committed golden vectors (tests/golden/*), made by make_golden.py
from the real reference.  Test infrastructure only."""

import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

_CACHE = {}


def load():
    if not _CACHE:
        _CACHE["arrays"] = dict(np.load(os.path.join(HERE, "golden.npz")))
        with open(os.path.join(HERE, "cases.json")) as fh:
            _CACHE["table"] = json.load(fh)
    return _CACHE["arrays"], _CACHE["table"]


def compress_cases():
    arrays, table = load()
    out = []
    for case in table["compress"]:
        p = f"c/{case['name']}/"
        c = dict(case)
        for key in ("input", "mask", "maxima", "indices", "coeffs", "decompressed"):
            c[key] = arrays[p + key]
        out.append(c)
    return out


def compress_case(name):
    return next(c for c in compress_cases() if c["name"] == name)


def op_cases():
    arrays, table = load()
    out = []
    for case in table["ops"]:
        p = f"o/{case['name']}/"
        c = dict(case)
        c["arrays"] = {k[len(p):]: v for k, v in arrays.items() if k.startswith(p)}
        out.append(c)
    return out


def float_ulps(a, b, kind):
    """|a-b| in units of the kind's ulp at b (finite entries)."""
    sig = {"bf16": 7, "f16": 10, "f32": 23, "f64": 52}[kind]
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    _, e = np.frexp(np.where(b == 0, 1.0, np.abs(b)))
    ulp = np.ldexp(1.0, e - 1 - sig)
    return np.abs(a - b) / ulp
