"""Dev: locate mismatches of a TMA config against the oracle (run with HARRIS_TMA_CONFIG=k)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402
from oracle import cref, synth  # noqa: E402

for (H, W) in [(5, 8), (6, 12), (9, 132), (13, 20), (37, 64), (64, 136), (100, 260), (133, 516), (300, 2564)]:
    rgb = synth.synth_numpy(3, H, W, seed=H * 1000 + W)
    for exact in (True, False):
        got = hb.harris(torch.from_numpy(rgb).cuda(), exact=exact).cpu().numpy()
        if exact:
            ref = cref.harris_f32(rgb)
            bad = np.argwhere(got != ref)
            msg = f"mismatch {len(bad)}/{ref.size}"
            if len(bad):
                r, c = bad[0]
                msg += f" first ({r},{c}) got {got[r, c]!r} ref {ref[r, c]!r} cols {sorted(set(bad[:, 1].tolist()))[:12]}"
        else:
            ok, m = synth.within_tolerance(got, cref.harris_f64(rgb))
            msg = f"tol ok={ok} {m}"
        print(H, W, "exact" if exact else "fast", msg, flush=True)
