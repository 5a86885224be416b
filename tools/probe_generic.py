"""Dev: device time of the generic (non-TMA) kernel vs the TMA path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402


def t(fn, iters=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    evs = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    return ts[len(ts) // 2]


for (B, H, W) in [(1, 8192, 8192), (1, 8190, 8190), (1, 8192, 8191), (64, 1080, 1918), (64, 1080, 1920)]:
    x = torch.empty((B, 3, H, W), device="cuda")
    hb.synth_(x.view(B * 3, H, W), seed=1)
    out = torch.empty((B, H - 4, W - 4), device="cuda")
    px = B * (H - 4) * (W - 4)
    nb = hb.algorithmic_bytes(H - 4, W - 4, B)
    for name, kw in (("auto", {}), ("generic", {"force_generic": True})):
        ms = t(lambda: hb.harris(x, out=out, **kw))
        print(f"{B}x{H}x{W} {name:8s} path={hb.context().last_path} {ms:.4f} ms {px / ms / 1e3:,.0f} MP/s "
              f"{nb / ms / 1e6:,.0f} GB/s")
    del x, out
    torch.cuda.empty_cache()
