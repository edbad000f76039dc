"""Run each hot-path op a few times on one workload (for ncu captures).

    ncu --set full -k regex:k_ -c 12 python tools/profile_ops.py c2
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import paper_2406_11209_b200 as bz  # noqa: E402
from quick_bench import CONFIGS, fill  # noqa: E402


def main(name, reps=2):
    shape, block, fk, ik, mask = CONFIGS[name]
    bits = (np.indices(block).sum(axis=0) <= 4) if mask == "lowpass" else None
    s = bz.CodecSettings(block, bz.FloatKind(fk), bz.IndexKind(ik),
                         mask=None if bits is None else bz.PruningMask(block, bits))
    kind = bz.FloatKind(fk)
    x = fill(shape, kind, 1)
    y = fill(shape, kind, 2)
    ca = bz.compress(x, s)
    cb = bz.compress(y, s)
    only = os.environ.get("PROFILE_ONLY")  # one op: l2 | dot | cov | mean
    if only:
        ops = {"l2": lambda: bz.ops.moments_record(ca, dc_only=2),
               "dot": lambda: bz.ops.moments_record(ca, cb, dc_only=2),
               "cov": lambda: bz.ops.moments_record(ca, cb),
               "mean": lambda: bz.ops.moments_record(ca, dc_only=True),
               "add": lambda: bz.add(ca, cb),
               "dec": lambda: bz.decompress(ca),
               "comp": lambda: bz.compress(x, s),
               "sub_l2": lambda: bz.ops._subtract_l2_sq(
                   ca, cb, torch.empty(1, dtype=torch.float64, device=ca.device))}
        for _ in range(reps):
            ops[only]()
        torch.cuda.synchronize()
        return
    for _ in range(reps):
        bz.compress(x, s)
        bz.decompress(ca)
        bz.decompress(ca, kind)
        bz.ops.moments_record(ca, dc_only=2)
        bz.ops.moments_record(ca, cb, dc_only=2)
        bz.ops.moments_record(ca, dc_only=True)
        bz.add(ca, cb)
        bz.negate(ca)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c2")
