"""Host-side latency of the scalar reductions (what a caller of l2_norm/mean waits).

    python tools/latency_probe.py [c2]

Prints wall-clock microseconds per call for: the fused kernel alone (device
time, CUDA events), the launch call alone (host time), the record readback,
the whole public call, and a cProfile of the public call.
"""

import cProfile
import os
import pstats
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import paper_2406_11209_b200 as bz  # noqa: E402
from paper_2406_11209_b200 import ops  # noqa: E402
from quick_bench import CONFIGS, fill, timeit  # noqa: E402


def wall(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


def main(name):
    shape, block, fk, ik, _ = CONFIGS[name]
    s = bz.CodecSettings(block, bz.FloatKind(fk), bz.IndexKind(ik))
    for shp in [(64,) * len(shape), shape]:
        x = fill(shp, bz.FloatKind(fk), 1)
        ca = bz.compress(x, s)
        rec = ops.moments_record(ca)
        print(f"== {name} {shp}")
        print(f"  kernel l2 (events)      {timeit(lambda: ops.moments_record(ca), 50) * 1e3:8.1f} us")
        print(f"  kernel dc (events)      {timeit(lambda: ops.moments_record(ca, dc_only=True), 50) * 1e3:8.1f} us")
        print(f"  launch only (host)      {wall(lambda: ops.moments_record(ca)):8.1f} us")
        tiny = torch.zeros(16, dtype=torch.int8, device="cuda")
        st = torch.cuda.current_stream()
        print(f"  bare stream sync        {wall(lambda: st.synchronize()):8.1f} us")
        print(f"  tiny launch + sync      {wall(lambda: (bz._native.call('bz_negate', 1, tiny.data_ptr(), tiny.data_ptr(), 16, st.cuda_stream), st.synchronize())):8.1f} us")
        print(f"  moments + sync          {wall(lambda: (ops.moments_record(ca, dc_only=2), st.synchronize())):8.1f} us")
        print(f"  record_to_host          {wall(lambda: ops.record_to_host(rec)):8.1f} us")
        print(f"  l2_norm (public)        {wall(lambda: bz.l2_norm(ca)):8.1f} us")
        print(f"  mean (public)           {wall(lambda: bz.mean(ca)):8.1f} us")
        print(f"  dot (public)            {wall(lambda: bz.dot(ca, ca)):8.1f} us")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        bz.l2_norm(ca)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)


def mean_breakdown(name="c3"):
    """Where mean(api) spends its time: the public call, the direct reduce,
    the two raw library calls, and the floor of one tiny launch + flag wait."""
    import ctypes
    shape, block, fk, ik, _ = CONFIGS[name]
    s = bz.CodecSettings(block, bz.FloatKind(fk), bz.IndexKind(ik))
    ca = bz.compress(fill(shape, bz.FloatKind(fk), 1), s)
    lib = bz._native.load_library()
    h = ops._host_record()
    hn = ops._host_record_np()
    La = ca.layout()
    ws = ops._reduce_workspace(ca.device, La)
    stream = bz._native.stream_handle(ca._dev_index)
    hp = h.data_ptr()

    def raw():
        hn[15] = 0.0
        lib.bz_moments_dc(ctypes.byref(La), ca.maxima.data_ptr(), ca._dc.data_ptr(), hp,
                          ws.data_ptr(), ws.numel(), stream)
        lib.bz_wait_record(ctypes.c_void_p(hp), ctypes.c_void_p(stream))

    def launch_only():
        lib.bz_moments_dc(ctypes.byref(La), ca.maxima.data_ptr(), ca._dc.data_ptr(), hp,
                          ws.data_ptr(), ws.numel(), stream)

    print(f"== mean breakdown {name}")
    print(f"  mean (public)           {wall(lambda: bz.mean(ca), 2000):8.1f} us")
    print(f"  _reduce_direct          {wall(lambda: ops._reduce_direct(ca, None, 1, h, hn), 2000):8.1f} us")
    print(f"  raw launch + wait       {wall(raw, 2000):8.1f} us")
    print(f"  raw launch only (host)  {wall(launch_only, 2000):8.1f} us")
    print(f"  plane kernel (events)   {timeit(lambda: ops.moments_record(ca, dc_only=1), 50) * 1e3:8.1f} us")



if __name__ == "__main__":
    if os.environ.get("MEAN_BREAKDOWN"):
        mean_breakdown(os.environ["MEAN_BREAKDOWN"])
    else:
        main(sys.argv[1] if len(sys.argv) > 1 else "c2")

