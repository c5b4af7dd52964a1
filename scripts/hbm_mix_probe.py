"""HBM rate of a read-only stream and of a device-to-device copy (the MEASURED_PEAKS.json recipe) on the same box:
context for roofline fractions above 1 of read-dominated kernels (A.V reads ~80 % of its bytes)."""
import torch

n = 1 << 31  # 4 GiB of bf16
a = torch.empty(n, dtype=torch.bfloat16, device="cuda").normal_()
b = torch.empty_like(a)
v = a.view(-1, 1 << 16)


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


ms = t(lambda: b.copy_(a))
print(f"copy: {2 * n * 2 / ms / 1e6:.0f} GB/s (read + write)")
ms = t(lambda: v.sum(dim=1, dtype=torch.float32))
print(f"read-only (row sums): {n * 2 / ms / 1e6:.0f} GB/s")
