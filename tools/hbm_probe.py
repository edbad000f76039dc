"""HBM read-only / write-only / copy bandwidth on this B200 (CUDA events),
to compare the write-heavy decompress kernels against a pure-write stream."""
import torch

n = 1 << 29  # 4 GiB per buffer
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n, dtype=torch.float64, device="cuda")
a.uniform_()


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


nb = n * 8
print(f"write (fill_)   {nb / t(lambda: b.fill_(1.0)) / 1e6:8.0f} GB/s")
print(f"read  (sum)     {nb / t(lambda: a.sum()) / 1e6:8.0f} GB/s")
print(f"copy  (copy_)   {2 * nb / t(lambda: b.copy_(a)) / 1e6:8.0f} GB/s")
