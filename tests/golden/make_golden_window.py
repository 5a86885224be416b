"""Golden fixtures for the Harris variant with the binomial window (PAPER.md:3937-3938:
the binomial filter "sometimes used as part of the Harris corner detection instead of the
3x3 '+' convolution").  Run in the build container (needs the reference package):

    python tests/golden/make_golden_window.py

Every output is the reference package's own evaluator (sges ``evalref.eval_term``) on the
thesis Harris Rise term with ``+3x3`` replaced by the reference's binomial stencil
``map (map (dot (join weights2d))) (3x3 neighbourhoods)`` (oracle/sges_oracle.py,
``harris_source("binomial")``; weights2d at evalref.py:114-115), in f64.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import sges_oracle, synth  # noqa: E402

CASES = [  # (H, W, seed, dist)
    (5, 5, 21, 0),
    (5, 9, 22, 1),
    (7, 12, 23, 2),
    (13, 17, 24, 0),
    (9, 132, 25, 1),   # crosses one 128-column warp strip
    (37, 64, 26, 0),
    (40, 52, 27, 2),
    (68, 140, 28, 0),
    (96, 96, synth.SEED, 0),
]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    if not sges_oracle.available():
        raise SystemExit("reference package not available")
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"generator": "sges.evalref.eval_term on the thesis Rise harris term with the binomial window "
                               "(oracle/sges_oracle.py harris_source('binomial'))",
                  "python": sys.version.split()[0], "term": sges_oracle.harris_source("binomial"), "cases": []}
    for H, W, seed, dist in CASES:
        name = f"binwin_{H}x{W}_s{seed}_d{dist}"
        rgb = synth.synth_numpy(3, H, W, seed=seed, dist=dist)
        t0 = time.time()
        out = sges_oracle.harris_sges(rgb, "binomial")
        dt = time.time() - t0
        arrays[name] = out
        meta["cases"].append({"name": name, "H": H, "W": W, "seed": seed, "dist": dist,
                              "input_sha256": sha(rgb), "output_sha256": sha(out),
                              "max_abs_ref": float(np.max(np.abs(out))), "sges_seconds": round(dt, 3)})
        print(name, f"{dt:.2f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "harris_binwin_golden.npz"), **arrays)
    with open(os.path.join(HERE, "harris_binwin_golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
