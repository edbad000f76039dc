"""Per-piece host cost of one public reduction call (mean / l2_norm), on a
small array so the GPU is idle: where the microseconds of the API go."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2406_11209_b200 as bz  # noqa: E402
from paper_2406_11209_b200 import _native, ops  # noqa: E402
from quick_bench import fill  # noqa: E402


def us(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


s = bz.CodecSettings((8, 8, 8), bz.FloatKind.F32, bz.IndexKind.I8)
a = bz.compress(fill((64, 64, 64), bz.FloatKind.F32, 1), s)
st = torch.cuda.current_stream()
h = ops._host_record()
La = a.layout()
ws = ops._reduce_workspace(a.device, La)
b = bz.compress(fill((64, 64, 64), bz.FloatKind.F32, 2), s)
print(f"mean (public)              {us(lambda: bz.mean(a)):7.2f} us")
print(f"covariance (public)        {us(lambda: bz.covariance(a, b)):7.2f} us")
print(f"ssim (public)              {us(lambda: bz.ssim(a, b)):7.2f} us")
print(f"dot (public)               {us(lambda: bz.dot(a, b)):7.2f} us")
print(f"_check_compatible          {us(lambda: ops._check_compatible(a, b)):7.2f} us")
print(f"l2_norm (public)           {us(lambda: bz.l2_norm(a)):7.2f} us")
print(f"_reduce(dc_only=1)         {us(lambda: ops._reduce(a, dc_only=True)):7.2f} us")
print(f"moments_record -> pinned   {us(lambda: ops.moments_record(a, dc_only=1, out=h)):7.2f} us")
print(f"  + stream sync            {us(lambda: (ops.moments_record(a, dc_only=1, out=h), st.synchronize())):7.2f} us")
print(f"raw ctypes bz_moments_dc   {us(lambda: _native.call('bz_moments_dc', __import__('ctypes').byref(La), a.maxima.data_ptr(), a.dc_plane.data_ptr(), h.data_ptr(), ws.data_ptr(), ws.numel(), st.cuda_stream)):7.2f} us")
lib = _native.load_library()
tiny = torch.zeros(16, dtype=torch.int8, device="cuda")
print(f"ctypes bz_version()        {us(lambda: lib.bz_version()):7.2f} us")
print(f"ctypes bz_negate launch    {us(lambda: lib.bz_negate(0, tiny.data_ptr(), tiny.data_ptr(), 16, st.cuda_stream)):7.2f} us")
print(f"ctypes bz_moments_dc bad L {us(lambda: lib.bz_moments_dc(None, 0, 0, 0, 0, 0, st.cuda_stream)):7.2f} us")
print(f"torch tiny kernel launch   {us(lambda: tiny.neg_()):7.2f} us")
mo = torch.empty_like(a.maxima)
import ctypes as _ct
print(f"ctypes bz_mul_scalar       {us(lambda: lib.bz_mul_scalar(_ct.byref(La), a.maxima.data_ptr(), a.indices.data_ptr(), None, 0.5, mo.data_ptr(), None, None, st.cuda_stream)):7.2f} us")
rec_d = torch.empty(16, dtype=torch.float64, device="cuda")
print(f"ctypes bz_moments_dc dev   {us(lambda: lib.bz_moments_dc(_ct.byref(La), a.maxima.data_ptr(), a.dc_plane.data_ptr(), rec_d.data_ptr(), ws.data_ptr(), ws.numel(), st.cuda_stream)):7.2f} us")
print(f"ctypes bz_moments sums     {us(lambda: lib.bz_moments(_ct.byref(La), _ct.byref(La), a.maxima.data_ptr(), a.indices.data_ptr(), None, None, 0, 2, rec_d.data_ptr(), ws.data_ptr(), ws.numel(), st.cuda_stream)):7.2f} us")
print(f"a.layout()                 {us(lambda: a.layout()):7.2f} us")
print(f"_reduce_workspace          {us(lambda: ops._reduce_workspace(a.device, La)):7.2f} us")
print(f"stream_handle              {us(lambda: _native.stream_handle(a.device)):7.2f} us")
print(f"current_stream()           {us(lambda: torch.cuda.current_stream(a.device)):7.2f} us")
print(f"Record.from_array          {us(lambda: ops.Record.from_array(h.numpy())):7.2f} us")
print(f"h.numpy()                  {us(lambda: h.numpy()):7.2f} us")
print(f"on_device wrapper (noop)   {us(lambda: _native.on_device(lambda x: x)(a)):7.2f} us")
print(f"bare st.synchronize        {us(lambda: st.synchronize()):7.2f} us")
print(f"data_ptr x2                {us(lambda: (a.maxima.data_ptr(), a.indices.data_ptr())):7.2f} us")
