"""Quick device-time probe of the fused kernel per TMA config (dev tool, not the bench).

python tools/probe_perf.py [--configs 0,1,2,3] [--iters 20]
Prints one line per (workload, config): ms, MP/s, algorithmic GB/s, fraction of
MEASURED_PEAKS.json hbm_gbs.  Inputs are larger than L2 (no flush needed).
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402


def peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        return 6650.0


def time_cfg(cfg, workloads, iters, exact=False, generic=False):
    env = dict(os.environ, HARRIS_DEV="1", HARRIS_TMA_CONFIG=str(cfg))
    code = f"""
import sys, torch, json
sys.path.insert(0, {ROOT!r})
import paper_2212_12035_b200 as hb
res = []
for (B, H, W) in {workloads!r}:
    x = torch.empty((B, 3, H, W), device='cuda')
    hb.synth_(x.view(B * 3, H, W), seed=12035)
    out = torch.empty((B, H - 4, W - 4), device='cuda')
    for _ in range(3):
        hb.harris(x, out=out, exact={exact}, force_generic={generic})
    torch.cuda.synchronize()
    evs = []
    for _ in range({iters}):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); hb.harris(x, out=out, exact={exact}, force_generic={generic}); e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    ms = ts[len(ts) // 2]
    info = hb.context().plan(H - 4, W - 4, B)
    res.append(dict(B=B, H=H, W=W, ms=ms, min_ms=ts[0], plan=info, path=hb.context().last_path))
    del x, out
    torch.cuda.empty_cache()
print(json.dumps(res))
"""
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    if r.returncode != 0:
        print(r.stderr[-2000:])
        return []
    return json.loads(r.stdout.strip().splitlines()[-1])


def time_u8(cfg, workloads, iters):
    env = dict(os.environ, HARRIS_DEV="1", HARRIS_U8_CONFIG=str(cfg))
    code = f"""
import sys, torch, json
sys.path.insert(0, {ROOT!r})
import paper_2212_12035_b200 as hb
res = []
g = torch.Generator(device='cuda'); g.manual_seed(12035)
for (B, H, W) in {workloads!r}:
    x = torch.randint(0, 256, (B, H, W, 3), dtype=torch.uint8, device='cuda', generator=g)
    out = torch.empty((B, H - 4, W - 4), device='cuda')
    for _ in range(3):
        hb.harris_u8(x, out=out)
    torch.cuda.synchronize()
    evs = []
    for _ in range({iters}):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); hb.harris_u8(x, out=out); e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    res.append(dict(B=B, H=H, W=W, ms=ts[len(ts) // 2], min_ms=ts[0], path=hb.context().last_path))
    del x, out
    torch.cuda.empty_cache()
print(json.dumps(res))
"""
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    if r.returncode != 0:
        print(r.stderr[-2000:])
        return []
    return json.loads(r.stdout.strip().splitlines()[-1])


def time_stencil(workloads, iters):
    code = f"""
import sys, torch, json
sys.path.insert(0, {ROOT!r})
import paper_2212_12035_b200 as hb
res = []
for (B, H, W) in {workloads!r}:
    x = torch.empty((B, H, W), device='cuda')
    hb.synth_(x, seed=12035)
    out = torch.empty((B, H - 2, W - 2), device='cuda')
    for _ in range(3):
        hb.stencil3x3_sep(x, out=out)
    torch.cuda.synchronize()
    evs = []
    for _ in range({iters}):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); hb.stencil3x3_sep(x, out=out); e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    res.append(dict(B=B, H=H, W=W, ms=ts[len(ts) // 2], min_ms=ts[0], path=hb.context().last_path))
    del x, out
    torch.cuda.empty_cache()
print(json.dumps(res))
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    if r.returncode != 0:
        print(r.stderr[-2000:])
        return []
    return json.loads(r.stdout.strip().splitlines()[-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,1,2,3")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--generic", action="store_true")
    ap.add_argument("--u8", action="store_true")
    ap.add_argument("--stencil", action="store_true")
    a = ap.parse_args()
    workloads = [(1, 8192, 8192), (1024, 1080, 1920), (1, 1536, 2560)]
    pk = peak()
    if a.stencil:
        for r in time_stencil(workloads, a.iters):
            B, H, W = r["B"], r["H"], r["W"]
            nbytes = B * (4 * H * W + 4 * (H - 2) * (W - 2))
            gbs = nbytes / (r["ms"] * 1e-3) / 1e9
            mps = B * (H - 2) * (W - 2) / (r["ms"] * 1e-3) / 1e6
            print(f"stencil3x3 {B}x{H}x{W}: {r['ms']:.4f} ms (min {r['min_ms']:.4f}) {mps:,.0f} MP/s "
                  f"{gbs:,.0f} GB/s frac={gbs / pk:.3f} path={r['path']}", flush=True)
        return
    if a.u8:
        for cfg in [int(c) for c in a.configs.split(",")]:
            for r in time_u8(cfg, workloads, a.iters):
                B, H, W = r["B"], r["H"], r["W"]
                nbytes = B * (3 * H * W + 4 * (H - 4) * (W - 4))
                gbs = nbytes / (r["ms"] * 1e-3) / 1e9
                mps = B * (H - 4) * (W - 4) / (r["ms"] * 1e-3) / 1e6
                print(f"u8 cfg{cfg} {B}x{H}x{W}: {r['ms']:.4f} ms (min {r['min_ms']:.4f}) {mps:,.0f} MP/s "
                      f"{gbs:,.0f} GB/s frac={gbs / pk:.3f} path={r['path']}", flush=True)
        return
    for cfg in [int(c) for c in a.configs.split(",")]:
        for r in time_cfg(cfg, workloads, a.iters, a.exact, a.generic):
            B, H, W = r["B"], r["H"], r["W"]
            nbytes = hb.algorithmic_bytes(H - 4, W - 4, B)
            gbs = nbytes / (r["ms"] * 1e-3) / 1e9
            mps = B * (H - 4) * (W - 4) / (r["ms"] * 1e-3) / 1e6
            print(f"cfg{cfg} exact={a.exact} generic={a.generic} {B}x{H}x{W}: {r['ms']:.4f} ms (min {r['min_ms']:.4f}) "
                  f"{mps:,.0f} MP/s {gbs:,.0f} GB/s frac={gbs / pk:.3f} path={r['path']} "
                  f"plan=bands{r['plan']['bands']}x{r['plan']['band_rows']} tiles={r['plan']['tiles']} "
                  f"grid={r['plan']['grid_ctas']}", flush=True)


if __name__ == "__main__":
    main()
