"""Dev: DRAM streaming ceilings for read/write mixes (torch kernels, inputs >> L2)."""
import torch

N = 1 << 30  # 4 GiB of f32 per tensor
a = torch.rand(N, device="cuda")
b = torch.rand(N, device="cuda")
c = torch.empty(N, device="cuda")
d = torch.empty(N // 3, device="cuda")


def t(fn, nbytes, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(nbytes * iters / (e0.elapsed_time(e1) * 1e-3) / 1e9)


print("read only (sum)            GB/s", t(lambda: a.sum(), 4 * N))
print("copy 1:1 (c.copy_(a))      GB/s", t(lambda: c.copy_(a), 8 * N))
print("2:1 (torch.add(a,b,out=c)) GB/s", t(lambda: torch.add(a, b, out=c), 12 * N))
x3 = a[: 3 * (N // 3)].view(3, N // 3)
print("3:1 (sum of 3 planes -> 1) GB/s", t(lambda: torch.sum(x3, dim=0, out=d), 16 * (N // 3)))
