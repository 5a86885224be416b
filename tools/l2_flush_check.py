"""Dev: does the bench's L2 flush (1 GiB write + 1 GiB read at normal priority) evict the
input lines an evict_last launch left behind?  For the small single-image extras, each
policy ctx runs flush -> launch N times.  Plain run: median CUDA-event time per policy.
Under `ncu --cache-control none --metrics dram__bytes_read.sum,... -k regex:strip_kernel`
the DRAM bytes each launch reads show whether its input came from L2 (bytes << 12*H*W).
    python tools/l2_flush_check.py [iters]
"""
import json
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2212_12035_b200 as hb  # noqa: E402
from paper_2212_12035_b200 import _lib  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
dev = torch.device("cuda", 0)
scratch = torch.empty(1 << 28, device=dev)
scratch2 = torch.empty(1 << 28, device=dev)


def flush():
    scratch.fill_(0.0)
    scratch2.sum()


res = {}
for H, W in [(1536, 2560), (2832, 4256)]:
    x = torch.empty((3, H, W), device=dev)
    hb.synth_(x, seed=12035)
    out = torch.empty((H - 4, W - 4), device=dev)
    for name, pol in [("evict_last", _lib.L2_EVICT_LAST), ("evict_normal", _lib.L2_EVICT_NORMAL)]:
        ctx = hb.HarrisContext(0, l2_policy=pol)
        for _ in range(5):
            hb.harris(x, out=out, ctx=ctx)
        ts = []
        for _ in range(iters):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            hb.harris(x, out=out, ctx=ctx)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        res[f"{H}x{W} {name}"] = {"us_median": ts[len(ts) // 2] * 1e3, "us_min": ts[0] * 1e3,
                                  "algorithmic_read_bytes": 12 * H * W}
print(json.dumps(res, indent=1))
