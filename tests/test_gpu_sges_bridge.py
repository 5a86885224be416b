"""The in-package drop-in boundary with the B200 kernels behind it.

`sges_bridge.register` / `register_binomial` put `harris` / `binomial` into the reference
type environment as polymorphic schemes (infer.py:190-196, 252-253) and into the
evaluator's ambient map (evalref.py:142-144) with their DEFAULT implementations — the
fused Harris kernel and the separable-stencil kernel on the B200.  Programs calling them
are parsed, typed and evaluated by the unmodified reference package (`sges`, from
/root/reference here or the pip-installed copy in baseline/_ref on the GPU box), and the
results are compared with the reference evaluating the thesis's full inlined Rise
programs (f64; binomial goal PAPER.md:3935-4016).
"""
import numpy as np
import pytest
import torch

from oracle import cref, sges_oracle, synth

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not sges_oracle.available(), reason="reference package sges not installed")]

hb = pytest.importorskip("paper_2212_12035_b200")
from paper_2212_12035_b200 import sges_bridge  # noqa: E402

SRC = sges_oracle.REFERENCE_SRC


def _env_rgb(H, W):
    sges_oracle._sges()  # puts the reference package on sys.path
    from sges import nat, types
    return {"rgb": types.data(types.array(nat.const(3), types.array(nat.const(H),
                              types.array(nat.const(W), types.scalar()))))}


def _env_img(name, H, W):
    sges_oracle._sges()
    from sges import nat, types
    return {name: types.data(types.array(nat.const(H), types.array(nat.const(W), types.scalar())))}


@pytest.mark.parametrize("H,W,seed,dist", [(9, 12, 1, 0), (20, 37, 2, 1), (41, 70, 3, 0), (64, 133, 4, 2)])
def test_ambient_harris_runs_the_fused_kernel(cuda_ctx, H, W, seed, dist):
    rgb = synth.synth_numpy(3, H, W, seed=seed, dist=dist)
    env, amb = _env_rgb(H, W), {"rgb": rgb.astype(np.float64).tolist()}
    sges_bridge.register(env, amb, reference_src=SRC)  # default impl = the B200 kernel
    term, val = sges_bridge.evaluate("harris rgb", env, amb, reference_src=SRC)
    got = np.asarray(val, dtype=np.float64)
    assert got.shape == (H - 4, W - 4)
    assert str(H - 4) in str(term.ty) and str(W - 4) in str(term.ty)
    # the value that crossed the boundary is the kernel's output, bit for bit
    direct = hb.harris(torch.from_numpy(rgb).cuda()).cpu().numpy()
    assert np.array_equal(got, direct.astype(np.float64))
    assert cuda_ctx.last_path != 0
    # and it meets the §8(d) tolerance against the reference evaluating the whole thesis program
    ok, m = synth.within_tolerance(got.astype(np.float32), sges_oracle.harris_sges(rgb))
    assert ok, m


def test_ambient_harris_inside_a_larger_program(cuda_ctx):
    """`harris` as one primitive of a bigger Rise term: the reference evaluator maps a
    lambda over the kernel's result (squares every coarsity value)."""
    H, W = 24, 31
    rgb = synth.synth_numpy(3, H, W, seed=9)
    env, amb = _env_rgb(H, W), {"rgb": rgb.astype(np.float64).tolist()}
    sges_bridge.register(env, amb, reference_src=SRC)
    _, val = sges_bridge.evaluate(r"map (map (\x. mul x x)) (harris rgb)", env, amb, reference_src=SRC)
    k = hb.harris(torch.from_numpy(rgb).cuda()).cpu().numpy().astype(np.float64)
    assert np.array_equal(np.asarray(val), k * k)


def test_ambient_binomial_runs_the_stencil_kernel(cuda_ctx):
    """`binomial` (the separated goal as one primitive) on the B200 vs the reference
    evaluating both the initial (2-D) and the separated goal programs.  u8-valued inputs
    make every partial sum an integer < 2^24, so the f32 kernel is exact."""
    rng = np.random.default_rng(11)
    for H, W in [(7, 9), (33, 70), (66, 131)]:
        img = rng.integers(0, 256, size=(H, W)).astype(np.float32)
        env, amb = _env_img("img", H, W), {"img": img.astype(np.float64).tolist()}
        sges_bridge.register_binomial(env, amb, reference_src=SRC)
        _, val = sges_bridge.evaluate("binomial img", env, amb, reference_src=SRC)
        got = np.asarray(val)
        assert np.array_equal(got, sges_oracle.binomial_sges(img, "separated"))
        assert np.array_equal(got, sges_oracle.binomial_sges(img, "initial"))
    # real-valued input: f32 kernel within 1e-6 relative of the f64 reference
    img = synth.synth_numpy(1, 40, 52, seed=3)[0]
    env, amb = _env_img("img", 40, 52), {"img": img.astype(np.float64).tolist()}
    sges_bridge.register_binomial(env, amb, reference_src=SRC)
    _, val = sges_bridge.evaluate("binomial img", env, amb, reference_src=SRC)
    ref = sges_oracle.binomial_sges(img, "separated")
    assert np.max(np.abs(np.asarray(val) - ref)) <= 1e-6 * np.max(np.abs(ref))


def test_ambient_composition_binomial_of_harris(cuda_ctx):
    """Both primitives in one program: `binomial (harris rgb)` — the reference type
    checker solves 3.(n+4).(m+4) -> n.m -> (n-2).(m-2) and the evaluator runs both
    kernels; equals the two kernels chained directly."""
    H, W = 30, 45
    rgb = synth.synth_numpy(3, H, W, seed=21)
    env, amb = _env_rgb(H, W), {"rgb": rgb.astype(np.float64).tolist()}
    sges_bridge.register(env, amb, reference_src=SRC)
    sges_bridge.register_binomial(env, amb, reference_src=SRC)
    term, val = sges_bridge.evaluate("binomial (harris rgb)", env, amb, reference_src=SRC)
    assert np.asarray(val).shape == (H - 6, W - 6)
    k = hb.harris(torch.from_numpy(rgb).cuda())
    chained = hb.stencil3x3_sep(k).cpu().numpy().astype(np.float64)
    assert np.array_equal(np.asarray(val), chained)


def test_degenerate_sizes_rejected_before_the_kernel(cuda_ctx):
    """The reference type checker solves ?m = -2 for a 3x5x2 input (nat.py:211-239); the
    bridge must reject it before anything reaches the C-ABI."""
    env, amb = _env_rgb(5, 2), {"rgb": np.zeros((3, 5, 2)).tolist()}
    sges_bridge.register(env, amb, reference_src=SRC)
    with pytest.raises(ValueError):
        sges_bridge.evaluate("harris rgb", env, amb, reference_src=SRC)
