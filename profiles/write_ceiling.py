"""HBM write ceiling on this box: torch fill_ / memset of the C2 output size
(4 GB), timed with CUDA events (reference point for K3 expand)."""
import torch

n = 40000 * 100000
buf = torch.empty(n, dtype=torch.uint8, device="cuda")
src = torch.empty(n // 8, dtype=torch.uint8, device="cuda")
dst = torch.empty(n // 8, dtype=torch.uint8, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


t = timeit(lambda: buf.fill_(7))
print(f"fill_ 4 GB: {t:.3f} ms  {n / t / 1e6:.0f} GB/s")
t = timeit(lambda: buf.zero_())
print(f"zero_ 4 GB: {t:.3f} ms  {n / t / 1e6:.0f} GB/s")
t = timeit(lambda: dst.copy_(src))
print(f"copy 0.5 GB: {t:.3f} ms  {2 * n / 8 / t / 1e6:.0f} GB/s (read+write)")
