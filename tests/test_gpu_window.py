"""GPU: Harris with the binomial window (HARRIS_FLAG_BINOMIAL_WINDOW) — the variant the thesis
names for its binomial rewrite goal ("sometimes used as part of the Harris corner detection
instead of the 3x3 '+' convolution"), weights2d = [1,2,1]^T [1,2,1]
(evalref.py:114-115).

* EXACT order on every kernel path equals the C f32 restatement (oracle_harris_f32_window)
  bit for bit; the C f64 restatement is pinned to the reference evaluator on the modified Rise
  term (tests/golden/harris_binwin_golden.*, test_oracle.py).
* FAST (shipped) order meets the §8(d) tolerance against the f64 reference (the goldens
  themselves, and the C f64 oracle at larger sizes), and is bit-identical between the packed
  dual-strip core (TMA config 6) and the scalar core (config 0).
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import cref, sges_oracle, synth

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_2212_12035_b200")
from paper_2212_12035_b200 import _lib  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _ctx_cfg(cfg):
    old = {k: os.environ.get(k) for k in ("HARRIS_DEV", "HARRIS_TMA_CONFIG")}
    os.environ.update(HARRIS_DEV="1", HARRIS_TMA_CONFIG=str(cfg))
    try:
        return hb.HarrisContext(0)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_window_goldens_every_path(cuda_ctx):
    meta = json.load(open(os.path.join(HERE, "harris_binwin_golden.json")))
    arrays = dict(np.load(os.path.join(HERE, "harris_binwin_golden.npz")))
    for case in meta["cases"]:
        rgb = synth.synth_numpy(3, case["H"], case["W"], seed=case["seed"], dist=case["dist"])
        ref32 = cref.harris_f32(rgb, window="binomial")
        gold = arrays[case["name"]]
        for kw in ({}, {"force_generic": True}):
            ex = hb.harris(_dev(rgb), exact=True, window="binomial", **kw)
            fast = hb.harris(_dev(rgb), window="binomial", **kw)
            torch.cuda.synchronize()
            assert np.array_equal(ex.cpu().numpy(), ref32), (case["name"], kw)
            ok, m = synth.within_tolerance(fast.cpu().numpy(), gold)
            assert ok, (case["name"], kw, m)
        W = case["W"]
        assert cuda_ctx.last_path == _lib.PATH_GENERIC
        hb.harris(_dev(rgb), window="binomial")
        assert cuda_ctx.last_path == (_lib.PATH_TMA if W % 4 == 0 else _lib.PATH_GENERIC)


@pytest.mark.parametrize("B,H,W", [(1, 9, 132), (1, 300, 2564), (3, 41, 388), (5, 21, 136), (2, 1080, 1920)])
def test_window_tma_configs_bitexact_and_identical(cuda_ctx, B, H, W):
    rgb = synth.synth_numpy(3 * B, H, W, seed=B * H + W, dist=2).reshape(B, 3, H, W)
    x = _dev(rgb if B > 1 else rgb[0])
    outs = {}
    for cfg in (0, 6):
        ctx = _ctx_cfg(cfg)
        ex = hb.harris(x, exact=True, window="binomial", ctx=ctx)
        outs[cfg] = hb.harris(x, window="binomial", ctx=ctx)
        torch.cuda.synchronize()
        assert ctx.last_path == _lib.PATH_TMA
        exn = ex.cpu().numpy().reshape(B, H - 4, W - 4)
        for b in range(B):
            assert np.array_equal(exn[b], cref.harris_f32(rgb[b], window="binomial")), (cfg, b)
    assert torch.equal(outs[0], outs[6])  # one FAST arithmetic on both cores
    fast = outs[6].cpu().numpy().reshape(B, H - 4, W - 4)
    for b in range(B):
        ok, m = synth.within_tolerance(fast[b], cref.harris_f64(rgb[b], window="binomial"))
        assert ok, (b, m)
    # the default-window kernel on the same input differs (the flag really switches the window)
    assert not torch.equal(hb.harris(x), outs[6])


def test_window_layouts_u8_host_and_bands(cuda_ctx):
    # layouts no TMA kernel of the window variant covers run the generic kernel, same bits in EXACT
    for H, W in [(40, 262), (41, 263), (72, 263)]:
        rgb = synth.synth_numpy(3, H, W, seed=H + W)
        ex = hb.harris(_dev(rgb), exact=True, window="binomial")
        torch.cuda.synchronize()
        assert cuda_ctx.last_path == _lib.PATH_GENERIC
        assert np.array_equal(ex.cpu().numpy(), cref.harris_f32(rgb, window="binomial"))
    # u8 ingest: equal to the planar path on byte/255
    rng = np.random.default_rng(7)
    hwc = rng.integers(0, 256, size=(2, 36, 70, 3), dtype=np.uint8)
    got = hb.harris_u8(torch.from_numpy(hwc).cuda(), exact=True, window="binomial").cpu().numpy()
    f32 = np.ascontiguousarray(hwc.transpose(0, 3, 1, 2)).astype(np.float32) / np.float32(255.0)
    for b in range(2):
        assert np.array_equal(got[b], cref.harris_f32(f32[b], window="binomial"))
    # host buffers through harris_run_host (pipelined H2D / kernel / D2H)
    rgb = synth.synth_numpy(3, 300, 516, seed=3)
    host = hb.harris(rgb, exact=True, window="binomial")
    assert np.array_equal(host, cref.harris_f32(rgb, window="binomial"))
    # multi-GPU decomposition: row bands with a 4-row halo reproduce the single launch
    from paper_2212_12035_b200 import shard
    x = _dev(synth.synth_numpy(3, 1000, 900, seed=5))
    full = hb.harris(x, window="binomial")
    parts = [hb.harris(shard.band_view(x, b), window="binomial") for b in shard.row_bands(996, 4)]
    assert torch.equal(torch.cat(parts, 0), full)


def test_window_fullsize_8192(cuda_ctx):
    H = W = 8192
    x = torch.empty((3, H, W), device="cuda")
    hb.synth_(x, seed=12035)
    ex = hb.harris(x, exact=True, window="binomial")
    fast = hb.harris(x, window="binomial")
    torch.cuda.synchronize()
    host = x.cpu().numpy()
    assert np.array_equal(ex.cpu().numpy(), cref.harris_f32(host, window="binomial"))
    ok, m = synth.within_tolerance(fast.cpu().numpy(), cref.harris_f64(host, window="binomial"))
    assert ok, m


@pytest.mark.skipif(not sges_oracle.available(), reason="reference package sges not installed")
def test_window_as_ambient_primitive(cuda_ctx):
    """`harris_binomial` registered in the reference type environment / evaluator with the GPU
    kernel behind it, against the reference evaluating the whole modified Rise program."""
    from paper_2212_12035_b200 import sges_bridge
    sges_oracle._sges()
    from sges import nat, types
    H, W = 24, 37
    rgb = synth.synth_numpy(3, H, W, seed=77)
    env = {"rgb": types.data(types.array(nat.const(3), types.array(nat.const(H),
                             types.array(nat.const(W), types.scalar()))))}
    amb = {"rgb": rgb.astype(np.float64).tolist()}
    src = sges_oracle.REFERENCE_SRC
    sges_bridge.register(env, amb, reference_src=src, name="harris_binomial", window="binomial")
    _, val = sges_bridge.evaluate("harris_binomial rgb", env, amb, reference_src=src)
    ok, m = synth.within_tolerance(np.asarray(val, np.float32), sges_oracle.harris_sges(rgb, "binomial"))
    assert ok, m
