"""Dev: host-side cost per call of the launch paths (no sync inside the loop; small image so
the GPU keeps up: numbers are host microseconds per call)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402
from paper_2212_12035_b200 import _lib  # noqa: E402

H, W = 68, 264
x = torch.empty((3, H, W), device="cuda")
hb.synth_(x, seed=1)
out = torch.empty((H - 4, W - 4), device="cuda")
ctx = hb.context(0)
L = _lib.lib()
st = torch.cuda.current_stream().cuda_stream
n, m = H - 4, W - 4


def per_call(fn, iters=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return round((t1 - t0) / iters * 1e6, 2)


xp, op = x.data_ptr(), out.data_ptr()
info = _lib.PlanInfo()
print("hb.harris(x, out=out)            us/call", per_call(lambda: hb.harris(x, out=out)))
print("ctx.run_strided (python method)  us/call",
      per_call(lambda: ctx.run_strided(op, m, n * m, n, m, xp, W, H * W, 3 * H * W, 1, 0.04, 0, st)))
print("L.harris_run_strided (raw ctypes) us/call",
      per_call(lambda: L.harris_run_strided(ctx.handle, op, m, n * m, n, m, xp, W, H * W, 3 * H * W, 1, 0.04, 0, st)))
print("L.harris_plan (no launch)        us/call",
      per_call(lambda: L.harris_plan(ctx.handle, n, m, 1, xp, W, H * W, 3 * H * W, op, m, n * m, 0, ctypes.byref(info))))
print("L.harris_abi_version (ctypes floor) us/call", per_call(lambda: L.harris_abi_version()))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    hb.harris(x, out=out)
print("CUDA graph replay                 us/call", per_call(lambda: g.replay()))
