"""Generate the golden fixtures that pin the oracle to the reference itself.

Run in the build container (needs /root/reference):

    python tests/golden/make_golden.py

For every case the Harris output is computed by the reference package's own
evaluator (sges ``evalref.eval_term`` on the thesis Rise program, see
``oracle/sges_oracle.py``) in f64.  Small cases store the full f64 output; the
512x512 config-1 case stores the SHA-256 of the f64 output bytes plus a crop,
because the C f64 oracle reproduces the evaluator bit-for-bit.

Synthetic inputs are regenerated from (seed, dist, shape) by
``oracle.synth.synth_numpy`` and checked against the stored input SHA-256;
hand-made inputs (smooth, constant, ramp, impulse) are stored verbatim.
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

SYNTH_CASES = [  # (H, W, seed, dist, full_output)
    (5, 5, 1, 0, True),
    (5, 9, 2, 1, True),
    (6, 7, 3, 0, True),
    (7, 9, 4, 1, True),
    (13, 17, 5, 0, True),
    (16, 16, 6, 1, True),
    (9, 132, 7, 0, True),     # crosses one 128-column warp strip
    (37, 64, 8, 0, True),
    (64, 64, 9, 1, True),
    (68, 140, 10, 0, True),
    (128, 128, synth.SEED, 0, True),
    (512, 512, synth.SEED, 0, False),  # config 1: hash only
]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def handmade() -> dict[str, np.ndarray]:
    H, W = 12, 20
    y = np.arange(H, dtype=np.float32)[:, None]
    x = np.arange(W, dtype=np.float32)[None, :]
    ramp = (0.01 * x + 0.02 * y).astype(np.float32)
    imp = np.zeros((3, 11, 11), dtype=np.float32)
    imp[:, 5, 5] = 1.0
    return {
        "constant": np.full((3, 9, 10), 0.375, dtype=np.float32),
        "ramp": np.stack([ramp, ramp, ramp]).astype(np.float32),
        "impulse": imp,
        "smooth": synth.smooth_image(40, 52),
    }


def main() -> None:
    if not sges_oracle.available():
        raise SystemExit("reference package not available")
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"generator": "sges.evalref.eval_term on the thesis Rise harris term "
                               "(oracle/sges_oracle.py)", "python": sys.version.split()[0],
                  "cases": []}
    for H, W, seed, dist, full in SYNTH_CASES:
        name = f"synth_{H}x{W}_s{seed}_d{dist}"
        rgb = synth.synth_numpy(3, H, W, seed=seed, dist=dist)
        t0 = time.time()
        out = sges_oracle.harris_sges(rgb)
        dt = time.time() - t0
        case = {"name": name, "kind": "synth", "H": H, "W": W, "seed": seed, "dist": dist,
                "input_sha256": sha(rgb), "output_sha256": sha(out),
                "max_abs_ref": float(np.max(np.abs(out))), "sges_seconds": round(dt, 3)}
        if full:
            arrays[name] = out
        else:
            arrays[name + "_crop"] = out[:16, :16].copy()
        meta["cases"].append(case)
        print(name, f"{dt:.2f}s", flush=True)
    for name, rgb in handmade().items():
        out = sges_oracle.harris_sges(rgb)
        arrays[name + "_input"] = rgb
        arrays[name] = out
        meta["cases"].append({"name": name, "kind": "stored", "H": rgb.shape[1], "W": rgb.shape[2],
                              "input_sha256": sha(rgb), "output_sha256": sha(out),
                              "max_abs_ref": float(np.max(np.abs(out)))})
    # drop-in boundary: harris as an ambient Rise primitive
    rgb = synth.synth_numpy(3, 9, 11, seed=11)
    via = sges_oracle.eval_via_ambient(rgb, lambda a: sges_oracle.harris_sges(a))
    meta["ambient_primitive_roundtrip_equal"] = bool(np.array_equal(via, sges_oracle.harris_sges(rgb)))
    np.savez_compressed(os.path.join(HERE, "harris_golden.npz"), **arrays)
    with open(os.path.join(HERE, "harris_golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
