"""Dev probe: small-image (configs[1]) device time with a clean L2 flush, per TMA config,
plus raw pinned H2D / D2H bandwidth (the ceiling of the e2e number)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

CODE = r"""
import sys, torch, json
sys.path.insert(0, ROOT)
import paper_2212_12035_b200 as hb
H, W = 1536, 2560
x = torch.empty((3, H, W), device='cuda'); hb.synth_(x, seed=12035)
out = torch.empty((H - 4, W - 4), device='cuda')
s1 = torch.empty(1 << 28, device='cuda'); s2 = torch.empty(1 << 28, device='cuda')
for _ in range(10): hb.harris(x, out=out)
evs = []
for _ in range(30):
    s1.fill_(0.0); s2.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); hb.harris(x, out=out); e1.record(); evs.append((e0, e1))
torch.cuda.synchronize()
ts = sorted(a.elapsed_time(b) for a, b in evs)
print(json.dumps(dict(ms=ts[len(ts)//2], min=ts[0], plan=hb.context().plan(H - 4, W - 4))))
"""


def main():
    for cfg in [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "0,3,6").split(",")]:
        env = dict(os.environ, HARRIS_DEV="1", HARRIS_TMA_CONFIG=str(cfg))
        r = subprocess.run([sys.executable, "-c", CODE.replace("ROOT", repr(ROOT))], env=env, capture_output=True,
                           text=True)
        print("cfg", cfg, r.stdout.strip()[-400:] or r.stderr[-400:], flush=True)
    # floor: the same byte volume as a plain copy (45 MB read + 15 MB written), same flush
    code = r"""
import torch
a = torch.empty(3 * 1536 * 2560, device='cuda'); b = torch.empty(1532 * 2556, device='cuda')
s1 = torch.empty(1 << 28, device='cuda'); s2 = torch.empty(1 << 28, device='cuda')
for _ in range(10): b.copy_(a[: b.numel()])
evs = []
for _ in range(30):
    s1.fill_(0.0); s2.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); a.sum(); b.copy_(a[: b.numel()]); e1.record(); evs.append((e0, e1))
torch.cuda.synchronize()
ts = sorted(x.elapsed_time(y) for x, y in evs)
print('copy-floor ms', ts[len(ts)//2], 'min', ts[0])
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-300:], flush=True)
    n = 4 << 30
    h = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
    d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(name, "GB/s", round(3 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1), flush=True)
    s2 = torch.cuda.Stream()
    h2 = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
    d2 = torch.empty(n // 4, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    print("bidirectional GB/s (each way)", round(n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1), flush=True)


if __name__ == "__main__":
    main()
