"""Golden records of the reference's oracle harness (bzc.metrics.compare_against_oracle,
metrics.py:224-323), from the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_oracle.py

Writes tests/golden/oracle_cmp.npz (the dense operands) and
tests/golden/oracle_cmp.json (one OpComparison record per case x operation).
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("BZC_REFERENCE_SRC", "/root/reference/pkg/src"))

import bzc  # noqa: E402
from bzc import metrics as bmetrics  # noqa: E402
from bzc.kinds import FloatKind, IndexKind  # noqa: E402

FK = {k.value: k for k in FloatKind}
IK = {k.value: k for k in IndexKind}

# name, shape, block, float kind, index kind, lowpass order (None = full), data
CASES = [
    ("f32_i8_3d", (16, 16, 24), (8, 8, 8), "f32", "i8", None, "normal"),
    ("f64_i16_2d", (20, 36), (4, 4), "f64", "i16", None, "uniform"),
    ("f32_i8_4d_lowpass", (8, 8, 8, 12), (4, 4, 4, 4), "f32", "i8", 4, "uniform"),
]
SCALARS = {"add_scalar": 0.75, "mul_scalar": -2.5}


def main():
    rng = np.random.default_rng(77)
    arrays, table = {}, []
    for name, shape, block, fk, ik, lowpass, dkind in CASES:
        bits = (np.ones(block, dtype=bool) if lowpass is None
                else np.indices(block).sum(axis=0) <= lowpass)
        s = bzc.CodecSettings(block, FK[fk], IK[ik], mask=bzc.PruningMask.from_bits(block, bits))
        xs = []
        for j in range(2):
            x = rng.normal(size=shape) if dkind == "normal" else rng.uniform(0, 1, size=shape)
            d = bzc.DenseArray.of(x, FK[fk])
            arrays[f"{name}/x{j}"] = np.asarray(d.values)
            xs.append(d)
        recs = {}
        for op, (arity, _kind) in bmetrics.ORACLE_OPERATIONS.items():
            c = bmetrics.compare_against_oracle(op, xs[:arity], s, x=SCALARS.get(op, 0.0))
            recs[op] = dataclasses.asdict(c)
        table.append({"name": name, "shape": list(shape), "block": list(block),
                      "float_kind": fk, "index_kind": ik, "lowpass": lowpass, "records": recs})
    np.savez_compressed(os.path.join(HERE, "oracle_cmp.npz"), **arrays)
    with open(os.path.join(HERE, "oracle_cmp.json"), "w") as fh:
        json.dump(table, fh, indent=1)
    print(f"{len(table)} cases -> tests/golden/oracle_cmp.npz, oracle_cmp.json")


if __name__ == "__main__":
    main()
