"""Dev: fixed launch overhead and copy floors around the configs[1] (1536x2560) launch.
All timings with an L2 flush (1 GiB write + 1 GiB read) before each timed op."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402

s1 = torch.empty(1 << 28, device="cuda")
s2 = torch.empty(1 << 28, device="cuda")


def flush():
    s1.fill_(0.0)
    s2.sum()


def timed(fn, iters=40):
    for _ in range(3):
        fn()
    evs = []
    for _ in range(iters):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in evs)
    return round(ts[len(ts) // 2], 2), round(ts[0], 2)


tiny_t = torch.empty(1, device="cuda")
print("minimal kernel (1-element fill_) after flush us", timed(lambda: tiny_t.fill_(1.0)))
xt = torch.empty((3, 12, 136), device="cuda")
hb.synth_(xt, seed=1)
ot = torch.empty((8, 132), device="cuda")
print("tiny harris 12x136 (fixed launch cost) us", timed(lambda: hb.harris(xt, out=ot)))
H, W = 1536, 2560
x = torch.empty((3, H, W), device="cuda")
hb.synth_(x, seed=12035)
out = torch.empty((H - 4, W - 4), device="cuda")
print("harris 1536x2560 us", timed(lambda: hb.harris(x, out=out)))
src = x.view(-1)
dst = torch.empty_like(src)
print("D2D copy 47 MB (read 47 + write 47) us", timed(lambda: dst.copy_(src)))
o2 = torch.empty_like(out)
print("read 47 MB + write 15.7 MB: sum + copy_ us", timed(lambda: (src.sum(), o2.copy_(out))))
print("write 15.7 MB only (fill_) us", timed(lambda: o2.fill_(1.0)))
print("read 47 MB only (sum) us", timed(lambda: src.sum()))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    hb.harris(x, out=out)
print("harris 1536x2560 via CUDA graph replay us", timed(lambda: g.replay()))
for n_img in (4, 16):
    xb = torch.empty((n_img, 3, H, W), device="cuda")
    hb.synth_(xb.view(-1, H, W), seed=12035)
    ob = torch.empty((n_img, H - 4, W - 4), device="cuda")
    t = timed(lambda: hb.harris(xb, out=ob), 20)
    print(f"harris batch {n_img}x1536x2560 us", t, "per image", round(t[0] / n_img, 2))
    del xb, ob
