"""mean through the DC plane at C3 (for ncu): compress two fields, the C3
chain, then mean three times."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2406_11209_b200 as bz  # noqa: E402
from quick_bench import CONFIGS, fill  # noqa: E402

shape, block, fk, ik, _ = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
s = bz.CodecSettings(block, bz.FloatKind(fk), bz.IndexKind(ik))
ca = bz.compress(fill(shape, bz.FloatKind(fk), 1), s)
cb = bz.compress(fill(shape, bz.FloatKind(fk), 2), s)
t = bz.mul_scalar(bz.add(ca, cb), 0.5)
for _ in range(3):
    print(bz.mean(t))
torch.cuda.synchronize()

# device time per call: 20 calls captured in a CUDA graph (no host launch cost)
from paper_2406_11209_b200 import ops  # noqa: E402


def graph_time(fn, n=20, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (n * reps) * 1e3


dev_rec = torch.empty(16, dtype=torch.float64, device="cuda")
host_rec = torch.empty(16, dtype=torch.float64, pin_memory=True)
strip = bz.CompressedArray(t.original_shape, t.settings, t.maxima, t.indices, _trusted=True)
print(f"plane -> device record   {graph_time(lambda: ops.moments_record(t, dc_only=1, out=dev_rec)):8.2f} us")
print(f"plane -> pinned record   {graph_time(lambda: ops.moments_record(t, dc_only=1, out=host_rec)):8.2f} us")
print(f"gather -> device record  {graph_time(lambda: ops.moments_record(strip, dc_only=1, out=dev_rec)):8.2f} us")
print(f"mul_scalar(0.5)          {graph_time(lambda: bz.mul_scalar(t, 0.5)):8.2f} us")
print(f"l2 sums -> device        {graph_time(lambda: ops.moments_record(t, dc_only=2, out=dev_rec)):8.2f} us")
