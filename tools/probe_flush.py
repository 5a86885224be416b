"""Dev: how the L2-flush size changes the measured cost of (a) a one-tile launch and
(b) the configs[1] image — separating cold-L2 cost from other after-flush effects."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402


def timed(fn, pre, iters=40):
    for _ in range(3):
        fn()
    evs = []
    for _ in range(iters):
        pre()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in evs)
    return round(ts[len(ts) // 2], 2)


xt = torch.empty((3, 12, 136), device="cuda")
hb.synth_(xt, seed=1)
ot = torch.empty((8, 132), device="cuda")
H, W = 1536, 2560
x = torch.empty((3, H, W), device="cuda")
hb.synth_(x, seed=12035)
out = torch.empty((H - 4, W - 4), device="cuda")
dummy = torch.empty(1 << 20, device="cuda")
tiny = lambda: hb.harris(xt, out=ot)  # noqa: E731
img = lambda: hb.harris(x, out=out)  # noqa: E731
print("no flush, previous op = tiny fill:", "tiny", timed(tiny, lambda: dummy.fill_(0)), "img", timed(img, lambda: dummy.fill_(0)))
for mb in (192, 256, 512, 1024, 4096):
    s1 = torch.empty(mb << 18, device="cuda")
    s2 = torch.empty(mb << 18, device="cuda")
    w = lambda: s1.fill_(0.0)  # noqa: E731
    wr = lambda: (s1.fill_(0.0), s2.sum())  # noqa: E731
    print(f"flush {mb} MB write: tiny {timed(tiny, w)} img {timed(img, w)} | write+read: tiny {timed(tiny, wr)} "
          f"img {timed(img, wr)} us")
    del s1, s2
    torch.cuda.empty_cache()
