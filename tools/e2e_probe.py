"""Where the end-to-end C2 step's time goes (bench.py e2e): per-step wall
time, H2D-only, and the step with the scalar read deferred."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_11209_b200 as bz  # noqa: E402

shape = (8192, 8192)
kind = bz.FloatKind.F64
s = bz.CodecSettings((4, 4), kind, bz.IndexKind.I16)
x = torch.randn(shape, dtype=torch.float64)
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
host_in = [x.pin_memory() for _ in streams]
host_out = [torch.empty(shape, dtype=torch.float64, pin_memory=True) for _ in streams]


def step(i, sync_l2=True):
    st = streams[i % 2]
    with torch.cuda.stream(st):
        a = bz.DenseArray(shape, kind, host_in[i % 2])
        c = bz.compress(a, s)
        rec = bz.ops.moments_record(c)
        if sync_l2:
            bz.l2_norm(c)
        out = bz.decompress(c)
        host_out[i % 2].copy_(out.values, non_blocking=True)
    return rec


for variant in ("bench", "deferred"):
    for i in range(3):
        step(i, variant == "bench")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 8
    for i in range(n):
        step(i, variant == "bench")
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n * 1e3
    print(f"{variant}: {dt:.2f} ms/step  {shape[0] * shape[1] * 8 / dt / 1e6:.1f} GB/s")

# H2D + D2H only
for i in range(3):
    with torch.cuda.stream(streams[i % 2]):
        d = host_in[i % 2].to("cuda", non_blocking=True)
        host_out[i % 2].copy_(d, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(8):
    with torch.cuda.stream(streams[i % 2]):
        d = host_in[i % 2].to("cuda", non_blocking=True)
        host_out[i % 2].copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"copies only: {(time.perf_counter() - t0) / 8 * 1e3:.2f} ms/step")
