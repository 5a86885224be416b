"""Golden fixtures for the separable 3x3 stencil row.

Run in the build container (needs /root/reference):

    python tests/golden/make_golden_binomial.py

Each case evaluates the reference package's binomial rewrite goal
with its own evaluator (``sges.evalref.eval_term``), both the initial program
(direct 2-D dot with weights2d) and the separated program (dot weightsV per column,
then dot weightsH), in f64.  Small cases store full outputs, the 256x256 case stores
SHA-256 hashes; inputs are regenerated from (seed, dist, shape) or stored (integer
image, on which every order and precision is exact).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import sges_oracle, synth  # noqa: E402

CASES = [(3, 3, 21, 0, True), (5, 9, 22, 1, True), (17, 23, 23, 0, True), (40, 130, 24, 0, True),
         (64, 64, 25, 1, True), (256, 256, 26, 0, False)]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    if not sges_oracle.available():
        raise SystemExit("reference package not available")
    arrays, meta = {}, {"generator": "sges.evalref.eval_term on the binomial goal programs "
                                     "(oracle/sges_oracle.py BINOMIAL_INITIAL / BINOMIAL_SEPARATED)",
                        "python": sys.version.split()[0], "cases": []}
    for H, W, seed, dist, full in CASES:
        name = f"binom_{H}x{W}_s{seed}_d{dist}"
        img = synth.synth_numpy(1, H, W, seed=seed, dist=dist)[0]
        case = {"name": name, "kind": "synth", "H": H, "W": W, "seed": seed, "dist": dist, "input_sha256": sha(img)}
        for form in ("initial", "separated"):
            out = sges_oracle.binomial_sges(img, form)
            case[f"{form}_sha256"] = sha(out)
            if full:
                arrays[f"{name}_{form}"] = out
        meta["cases"].append(case)
        print(name, flush=True)
    rng = np.random.default_rng(7)
    img = rng.integers(0, 256, size=(33, 47)).astype(np.float32)   # exact in every order
    arrays["binom_int_input"] = img
    case = {"name": "binom_int", "kind": "stored", "H": 33, "W": 47, "input_sha256": sha(img)}
    for form in ("initial", "separated"):
        out = sges_oracle.binomial_sges(img, form)
        arrays[f"binom_int_{form}"] = out
        case[f"{form}_sha256"] = sha(out)
    meta["cases"].append(case)
    np.savez_compressed(os.path.join(HERE, "binomial_golden.npz"), **arrays)
    json.dump(meta, open(os.path.join(HERE, "binomial_golden.json"), "w"), indent=1)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
