"""CPU: pin the separable-3x3 oracle to the reference's binomial goal.

The C f64 restatement reproduces the reference evaluator BIT-FOR-BIT for both the
initial (direct 2-D) and the separated (vertical-then-horizontal) program on every
committed fixture; the f32 order is within tolerance, and exact on integer images.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import cref, sges_oracle, synth

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def bgolden():
    meta = json.load(open(os.path.join(HERE, "binomial_golden.json")))
    return meta, dict(np.load(os.path.join(HERE, "binomial_golden.npz")))


def _img(case, arrays):
    if case["kind"] == "synth":
        img = synth.synth_numpy(1, case["H"], case["W"], seed=case["seed"], dist=case["dist"])[0]
    else:
        img = arrays["binom_int_input"]
    assert hashlib.sha256(np.ascontiguousarray(img).tobytes()).hexdigest() == case["input_sha256"]
    return img


def test_binomial_f64_bitexact_both_forms(oracle_lib, bgolden):
    meta, arrays = bgolden
    for case in meta["cases"]:
        img = _img(case, arrays)
        for form, fi in (("initial", 0), ("separated", 1)):
            out = cref.sep3x3_f64(img, form=fi)
            assert hashlib.sha256(out.tobytes()).hexdigest() == case[f"{form}_sha256"], (case["name"], form)


def test_binomial_f32_tolerance_and_integer_exactness(oracle_lib, bgolden):
    meta, arrays = bgolden
    for case in meta["cases"]:
        img = _img(case, arrays)
        ref = cref.sep3x3_f64(img)
        got = cref.sep3x3_f32(img)
        # stencil tolerance: normalised L-inf <= 1e-6 (f32 rounding of a 9-term weighted sum;
        # the Harris PSNR criterion is specific to coarsity magnitudes)
        assert synth.norm_linf(got, ref) <= 1e-6, case["name"]
    img = arrays["binom_int_input"]
    assert np.array_equal(cref.sep3x3_f32(img), arrays["binom_int_separated"])
    assert np.array_equal(cref.sep3x3_f32(img), arrays["binom_int_initial"])


def test_sep3x3_general_weights(oracle_lib):
    img = synth.synth_numpy(1, 30, 41, seed=9)[0]
    wv, wh = (0.25, 0.5, 0.25), (-1.0, 0.0, 1.0)
    direct = np.zeros((28, 39))
    for i in range(3):
        for j in range(3):
            direct += wv[i] * wh[j] * img[i:i + 28, j:j + 39].astype(np.float64)
    assert np.allclose(cref.sep3x3_f64(img, wv, wh, form=1), direct, rtol=0, atol=1e-12)
    assert np.allclose(cref.sep3x3_f32(img, wv, wh), direct, rtol=0, atol=1e-6)


@pytest.mark.skipif(not sges_oracle.available(), reason="/root/reference not present")
def test_binomial_live_reference(oracle_lib):
    img = synth.synth_numpy(1, 11, 14, seed=123)[0]
    assert np.array_equal(sges_oracle.binomial_sges(img, "initial"), cref.sep3x3_f64(img, form=0))
    assert np.array_equal(sges_oracle.binomial_sges(img, "separated"), cref.sep3x3_f64(img, form=1))


@pytest.mark.skipif(not sges_oracle.available(), reason="/root/reference not present")
def test_bridge_registers_binomial(oracle_lib):
    from paper_2212_12035_b200 import sges_bridge
    from sges import nat, types
    img = synth.synth_numpy(1, 9, 12, seed=5)[0]
    env = {"img": types.data(types.array(nat.const(9), types.array(nat.const(12), types.scalar())))}
    amb = {"img": img.astype(np.float64).tolist()}
    sges_bridge.register_binomial(env, amb, impl=lambda a: cref.sep3x3_f64(a, form=1),
                                  reference_src=sges_oracle.REFERENCE_SRC)
    term, val = sges_bridge.evaluate("binomial img", env, amb, reference_src=sges_oracle.REFERENCE_SRC)
    assert np.array_equal(np.asarray(val), sges_oracle.binomial_sges(img, "separated"))
