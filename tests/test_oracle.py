"""CPU: pin the oracle to the reference before trusting it (no GPU needed).

* The C f64 restatement reproduces the reference package's own evaluator
  (sges ``eval_term`` on the thesis Rise term) BIT-FOR-BIT on every committed
  golden fixture, including the 512x512 config-1 image (SHA-256 of the output).
* The C f32 restatement (Appendix-B op order, the GPU's exact mode) equals the
  independent numpy restatement bit-for-bit and sits within the SURVEY.md §8(d)
  tolerance of the f64 reference.
* When /root/reference is present (build container), the reference evaluator is
  also run live on fresh seeds.
"""
import hashlib

import numpy as np
import pytest

from oracle import cref, npref, sges_oracle, synth


def _input(case, arrays):
    if case["kind"] == "synth":
        rgb = synth.synth_numpy(3, case["H"], case["W"], seed=case["seed"], dist=case["dist"])
    else:
        rgb = arrays[case["name"] + "_input"]
    assert hashlib.sha256(np.ascontiguousarray(rgb).tobytes()).hexdigest() == case["input_sha256"]
    return rgb


def test_golden_f64_bitexact(oracle_lib, golden):
    meta, arrays = golden
    assert len(meta["cases"]) >= 14
    for case in meta["cases"]:
        rgb = _input(case, arrays)
        out = cref.harris_f64(rgb)
        assert out.shape == (case["H"] - 4, case["W"] - 4)
        assert hashlib.sha256(out.tobytes()).hexdigest() == case["output_sha256"], case["name"]
        if case["name"] in arrays:
            assert np.array_equal(out, arrays[case["name"]])
        else:
            assert np.array_equal(out[:16, :16], arrays[case["name"] + "_crop"])


def test_golden_f32_within_tolerance(oracle_lib, golden):
    meta, arrays = golden
    for case in meta["cases"]:
        rgb = _input(case, arrays)
        ok, m = synth.within_tolerance(cref.harris_f32(rgb), cref.harris_f64(rgb))
        assert ok, (case["name"], m)


def test_rrot_within_tolerance_on_goldens(oracle_lib, golden):
    """The thesis cbuf+rrot CPU schedule (a timed CPU baseline variant)
    against the f64 oracle that is pinned bit-for-bit to the reference evaluator, on every
    golden case incl. the 512^2 config-1 image."""
    meta, arrays = golden
    for case in meta["cases"]:
        rgb = _input(case, arrays)
        ok, m = synth.within_tolerance(cref.harris_f32_rrot(rgb), cref.harris_f64(rgb))
        assert ok, (case["name"], m)


@pytest.mark.parametrize("H,W,dist", [(5, 5, 0), (6, 11, 1), (31, 45, 2), (64, 130, 1), (203, 77, 0), (100, 517, 2)])
def test_rrot_c_equals_numpy_restatement(oracle_lib, H, W, dist):
    """oracle_harris_f32_rrot (line buffers, 32-row strips, register rotation) equals an
    independent whole-plane numpy restatement of the same arithmetic bit-for-bit, and is
    invariant to the thread count and to batching."""
    rgb = synth.synth_numpy(3, H, W, seed=3 * H + W, dist=dist)
    one = cref.harris_f32_rrot(rgb, nthreads=1)
    assert np.array_equal(one, npref.harris_rrot_np(rgb))
    assert np.array_equal(one, cref.harris_f32_rrot(rgb, nthreads=4))
    ok, m = synth.within_tolerance(one, cref.harris_f64(rgb))
    assert ok, m
    batch = np.stack([rgb, rgb[::-1].copy()])
    both = cref.harris_batched(batch, variant="rrot")
    assert np.array_equal(both[0], one) and np.array_equal(both[1], cref.harris_f32_rrot(batch[1]))


def test_ambient_primitive_recorded(golden):
    meta, _ = golden
    assert meta["ambient_primitive_roundtrip_equal"] is True


@pytest.mark.parametrize("H,W,dist", [(5, 5, 0), (6, 11, 1), (31, 45, 0), (64, 130, 1), (203, 77, 0)])
def test_c_f32_equals_numpy_f32(oracle_lib, H, W, dist):
    rgb = synth.synth_numpy(3, H, W, seed=H + W, dist=dist)
    assert np.array_equal(cref.harris_f32(rgb), npref.harris_np(rgb, dtype=np.float32))


@pytest.mark.parametrize("H,W", [(40, 52), (300, 211)])
def test_smooth_stress_tolerance(oracle_lib, H, W):
    rgb = synth.smooth_image(H, W)
    ok, m = synth.within_tolerance(cref.harris_f32(rgb), cref.harris_f64(rgb))
    assert ok, m


def test_thread_count_invariance(oracle_lib):
    rgb = synth.synth_numpy(3, 301, 257, seed=5)
    a = cref.harris_f32(rgb, nthreads=1)
    b = cref.harris_f32(rgb, nthreads=4)
    assert np.array_equal(a, b)


def test_synth_c_matches_numpy(oracle_lib):
    for dist in (0, 1):
        a = cref.synth(5, 40, 37, seed=12035, dist=dist, row0=7, rows=11, plane0=2, H_global=40)
        b = synth.synth_numpy(5, 40, 37, seed=12035, dist=dist, row0=7, rows=11, plane0=2, H_global=40)
        assert np.array_equal(a, b)
        full = synth.synth_numpy(7, 40, 37, seed=12035, dist=dist)
        assert np.array_equal(full[2:7, 7:18], b)
    u = synth.synth_numpy(3, 64, 64, seed=1)
    assert u.min() >= 0.0 and u.max() < 1.0
    q = synth.synth_numpy(3, 64, 64, seed=1, dist=1)
    assert np.array_equal(np.round(q * 255), q * 255) or np.allclose(np.round(q * 255), q * 255, atol=1e-4)


def test_oracle_rejects_small():
    with pytest.raises(ValueError):
        cref.harris_f32(np.zeros((3, 4, 9), np.float32))
    with pytest.raises(ValueError):
        npref.harris_np(np.zeros((3, 9, 4), np.float32))


def test_ramp_and_constant_known_answers(oracle_lib):
    a, b = 0.01, 0.02
    y = np.arange(24, dtype=np.float64)[:, None]
    x = np.arange(36, dtype=np.float64)[None, :]
    g = (a * x + b * y).astype(np.float32)
    out = cref.harris_f64(np.stack([g, g, g]))
    assert np.allclose(out, -0.64 * (a * a + b * b) ** 2, rtol=1e-4)
    assert np.all(cref.harris_f64(np.full((3, 9, 9), 0.7, np.float32)) == 0.0)


needs_ref = pytest.mark.skipif(not sges_oracle.available(), reason="/root/reference not present")


@needs_ref
@pytest.mark.parametrize("H,W,seed", [(6, 9, 101), (17, 23, 202)])
def test_live_reference_evaluator(oracle_lib, H, W, seed):
    rgb = synth.synth_numpy(3, H, W, seed=seed)
    assert np.array_equal(sges_oracle.harris_sges(rgb), cref.harris_f64(rgb))


@needs_ref
def test_live_reference_types_and_ambient_boundary():
    term, ty = sges_oracle.typed_term()
    assert "n" in str(ty) and "m" in str(ty)
    rgb = synth.synth_numpy(3, 9, 12, seed=3)
    via = sges_oracle.eval_via_ambient(rgb, cref.harris_f64)
    assert np.array_equal(via, sges_oracle.harris_sges(rgb))


@needs_ref
def test_sges_bridge_registration_types_and_evaluates(oracle_lib):
    """The product-side bridge registers `harris` with the reference type checker; here
    the implementation is the oracle (no GPU in this container) — on a GPU box with the
    reference installed the default implementation is the fused kernel."""
    from paper_2212_12035_b200 import sges_bridge
    from sges import types, nat
    rgb = synth.synth_numpy(3, 8, 10, seed=17)
    env = {"rgb": types.data(types.array(nat.const(3), types.array(nat.const(8),
                             types.array(nat.const(10), types.scalar()))))}
    amb = {"rgb": rgb.astype(np.float64).tolist()}
    sges_bridge.register(env, amb, impl=cref.harris_f64, reference_src=sges_oracle.REFERENCE_SRC)
    term, val = sges_bridge.evaluate("harris rgb", env, amb, reference_src=sges_oracle.REFERENCE_SRC)
    assert "4" in str(term.ty) and "6" in str(term.ty)
    assert np.array_equal(np.asarray(val), sges_oracle.harris_sges(rgb))
    bad = {"rgb": types.data(types.array(nat.const(3), types.array(nat.const(5),
                             types.array(nat.const(2), types.scalar()))))}
    amb_bad = {"rgb": np.zeros((3, 5, 2)).tolist()}
    sges_bridge.register(bad, amb_bad, impl=cref.harris_f64, reference_src=sges_oracle.REFERENCE_SRC)
    with pytest.raises(ValueError):
        sges_bridge.evaluate("harris rgb", bad, amb_bad, reference_src=sges_oracle.REFERENCE_SRC)


def test_opencv_composition_meets_tolerance(oracle_lib):
    """The thesis's OpenCV-composed comparison pipeline, restated with
    the image's OpenCV, matches the f64 oracle within the SURVEY.md §8(d) tolerance (it is a
    reported CPU baseline in bench.py)."""
    from oracle import cref, opencv_ref, synth
    if not opencv_ref.available():
        pytest.skip("cv2 not importable")
    for H, W, seed in [(64, 96, 1), (300, 517, 2)]:
        x = cref.synth(3, H, W, seed=seed)
        ok, m = synth.within_tolerance(opencv_ref.harris_opencv(x), cref.harris_f64(x))
        assert ok, m


# ---- Harris with the binomial window, pinned to the reference evaluator
def _binwin_golden():
    import json
    import os
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    meta = json.load(open(os.path.join(here, "harris_binwin_golden.json")))
    return meta, dict(np.load(os.path.join(here, "harris_binwin_golden.npz")))


def test_binomial_window_f64_bitexact_vs_reference_goldens(oracle_lib):
    meta, arrays = _binwin_golden()
    assert len(meta["cases"]) >= 9 and "weights2d" in meta["term"]
    for case in meta["cases"]:
        rgb = synth.synth_numpy(3, case["H"], case["W"], seed=case["seed"], dist=case["dist"])
        assert hashlib.sha256(rgb.tobytes()).hexdigest() == case["input_sha256"]
        out = cref.harris_f64(rgb, window="binomial")
        assert np.array_equal(out, arrays[case["name"]]), case["name"]
        assert hashlib.sha256(out.tobytes()).hexdigest() == case["output_sha256"]
        # the f32 restatement (the GPU's EXACT order) within the §8(d) tolerance, and equal to
        # the independent numpy restatement bit for bit
        f32 = cref.harris_f32(rgb, window="binomial")
        ok, m = synth.within_tolerance(f32, out)
        assert ok, (case["name"], m)
        assert np.array_equal(f32, npref.harris_np(rgb, dtype=np.float32, window="binomial")), case["name"]
    # the window changes the result (not the box sums under another name)
    rgb = synth.synth_numpy(3, 20, 30, seed=1)
    assert not np.allclose(cref.harris_f64(rgb, window="binomial"), cref.harris_f64(rgb))


@needs_ref
def test_binomial_window_live_reference(oracle_lib):
    rgb = synth.synth_numpy(3, 11, 19, seed=404, dist=2)
    assert np.array_equal(sges_oracle.harris_sges(rgb, "binomial"), cref.harris_f64(rgb, window="binomial"))
