"""Host cost per call of the launch paths (no synchronisation inside the loop; tiny images so the
GPU never backs the queue up).  python tools/host_overhead.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402
from paper_2212_12035_b200 import _lib  # noqa: E402

L = _lib.lib()
ctx = hb.context(0)
x = torch.rand(3, 12, 136, device="cuda")
out = torch.empty(8, 132, device="cuda")
x8 = torch.randint(0, 256, (12, 136, 3), dtype=torch.uint8, device="cuda")
out8 = torch.empty(8, 132, device="cuda")
info = _lib.PlanInfo()
st = torch.cuda.current_stream().cuda_stream


def per_call(fn, n=400):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / n * 1e6


rows = {
    "ctypes floor (harris_abi_version)": lambda: L.harris_abi_version(),
    "harris_plan (no launch)": lambda: L.harris_plan(ctx.handle, 8, 132, 1, x.data_ptr(), 136, 12 * 136, 3 * 12 * 136,
                                                    out.data_ptr(), 132, 8 * 132, 0, ctypes.byref(info)),
    "raw harris_run_strided": lambda: L.harris_run_strided(ctx.handle, out.data_ptr(), 132, 8 * 132, 8, 132, x.data_ptr(),
                                                          136, 12 * 136, 3 * 12 * 136, 1, 0.04, 0, st),
    "raw harris_run_u8": lambda: L.harris_run_u8(ctx.handle, out8.data_ptr(), 132, 8 * 132, 8, 132, x8.data_ptr(),
                                                 3 * 136, 12 * 3 * 136, 1, 0.04, 0, st),
    "hb.harris(x, out=out)": lambda: hb.harris(x, out=out),
    "hb.harris_u8(x8, out=out8)": lambda: hb.harris_u8(x8, out=out8),
    "torch out.zero_() (a torch launch, for scale)": lambda: out.zero_(),
}
for k, fn in rows.items():
    print(f"{k:48s} {per_call(fn):7.2f} us/call")
