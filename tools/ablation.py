"""Kernel-grouping ablation on B200.

python tools/ablation.py [--size 8192] [--iters 20] [--out profiles/ablation_rNN.json]

For each thesis grouping — [Sx],[Sy],[x],[+],[coarsity] / [Sx,Sy,x],[+,coarsity] /
[Sx,Sy],[x,+,coarsity] / fully fused — times one image (CUDA events, back-to-back,
median), checks the result against the fused exact kernel bit-for-bit, and reports the
compulsory HBM bytes of that grouping, so the fusion win is measured in bytes and time.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=8192)
    ap.add_argument("--width", type=int, default=None)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    H, W = a.size, a.width or a.size
    n, m = H - 4, W - 4
    x = torch.empty((3, H, W), device="cuda")
    hb.synth_(x, seed=12035)
    ref = hb.harris(x, exact=True)
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    res = {"image": [H, W], "peak_gbs": peak, "groupings": []}
    L = hb._lib.lib()
    for g in (1, 2, 3, 4):
        need = int(L.harris_grouping_scratch_bytes(g, n, m))
        scratch = torch.empty(max(need // 4, 1), device="cuda")
        out = torch.empty((n, m), device="cuda")
        for exact in (True, False) if g == 4 else (True,):
            fn = lambda: hb.harris_grouping(x, g, out=out, scratch=scratch, exact=exact)  # noqa: E731
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            same = bool(torch.equal(out, ref)) if exact else None
            evs = []
            for _ in range(a.iters):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                evs.append((e0, e1))
            torch.cuda.synchronize()
            ts = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
            ms = ts[len(ts) // 2]
            hbm = hb.grouping_hbm_bytes(g, n, m)
            row = {"grouping": g, "groups": hb.GROUPINGS[g], "kernels": int(L.harris_grouping_launches(g)),
                   "order": "exact" if exact else "fast", "ms_median": ms, "ms_min": ts[0],
                   "mp_per_s": n * m / (ms * 1e-3) / 1e6, "compulsory_hbm_bytes": hbm,
                   "bytes_per_output_px": hbm / (n * m), "hbm_gbs_at_compulsory": hbm / (ms * 1e-3) / 1e9,
                   "bit_identical_to_fused_exact": same}
            res["groupings"].append(row)
            print(json.dumps(row), flush=True)
        del scratch, out
        torch.cuda.empty_cache()
    fused = [r for r in res["groupings"] if r["grouping"] == 4 and r["order"] == "fast"][0]
    for r in res["groupings"]:
        r["fused_speedup"] = r["ms_median"] / fused["ms_median"]
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
