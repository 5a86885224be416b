"""Thesis CPU schedules on this host: cbuf vs cbuf+rrot (the thesis reports
rrot 1.24x faster than cbuf on its ARM CPU) at 1..all threads on a batch of
1080p images, plus one 8192^2 image.  MP/s of output pixels, best of 3 timed passes.
    python tools/cpu_schedules.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import cref  # noqa: E402


def mps(x, variant, threads, passes=3):
    out = np.zeros((x.shape[0], x.shape[2] - 4, x.shape[3] - 4), np.float32)
    cref.harris_batched(x, variant=variant, nthreads=threads, out=out)
    best = float("inf")
    for _ in range(passes):
        t0 = time.perf_counter()
        cref.harris_batched(x, variant=variant, nthreads=threads, out=out)
        best = min(best, time.perf_counter() - t0)
    return x.shape[0] * (x.shape[2] - 4) * (x.shape[3] - 4) / best / 1e6


ncpu = os.cpu_count() or 1
res = {"cpu_model": open("/proc/cpuinfo").read().split("model name")[1].split(":")[1].split("\n")[0].strip(),
       "threads_available": ncpu, "rows": []}
batch = cref.synth(3 * 32, 1080, 1920, seed=12035).reshape(32, 3, 1080, 1920)
big = cref.synth(3, 8192, 8192, seed=12035).reshape(1, 3, 8192, 8192)
for name, x in (("32 x 1080x1920", batch), ("8192x8192", big)):
    for t in sorted({1, 2, 4, 8, ncpu}):
        c, r = mps(x, "cbuf", t), mps(x, "rrot", t)
        row = {"workload": name, "threads": t, "cbuf_mps": c, "rrot_mps": r, "rrot_over_cbuf": r / c}
        res["rows"].append(row)
        print(json.dumps(row), flush=True)
print(json.dumps(res))
