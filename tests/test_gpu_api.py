"""GPU tests of the round-2 API surface: harris_init_ex options, the HARRIS_DEV gate on
developer knobs, and the argument validation of the Python wrappers."""
import ctypes
import os

import numpy as np
import pytest
import torch

from oracle import cref, synth

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_2212_12035_b200")
from paper_2212_12035_b200 import _lib  # noqa: E402

# f32 layouts covering every kernel path whose input loads carry an L2 policy hint:
# TMA (W % 4 == 0), pair-row TMA (W % 4 == 2), quad-row TMA (odd W, H % 4 == 0),
# bulk-copy K1b (odd W, H % 4 != 0)
LAYOUTS = [(70, 260), (70, 262), (72, 263), (71, 263)]


@pytest.mark.parametrize("policy", [_lib.L2_EVICT_FIRST, _lib.L2_EVICT_NORMAL, _lib.L2_EVICT_LAST])
def test_l2_policy_option_bit_identical(cuda_ctx, policy):
    ctx = hb.HarrisContext(0, l2_policy=policy)
    for H, W in LAYOUTS:
        rgb = torch.from_numpy(synth.synth_numpy(3, H, W, seed=H + W)).cuda()
        a = hb.harris(rgb, ctx=ctx, exact=True)
        b = hb.harris(rgb, ctx=ctx)
        torch.cuda.synchronize()
        ref = cref.harris_f32(rgb.cpu().numpy())
        assert np.array_equal(a.cpu().numpy(), ref), (H, W, ctx.last_path)
        assert torch.equal(b, hb.harris(rgb)), (H, W)  # FAST identical to the default-policy ctx


def test_init_ex_rejects_bad_options():
    L = _lib.lib()
    o = _lib.Options()
    L.harris_options_default(ctypes.byref(o))
    assert o.struct_size == ctypes.sizeof(_lib.Options) and o.l2_policy == _lib.L2_EVICT_LAST and o.band_rows == 0
    assert o.pdl == 1
    for field, val in [("l2_policy", 3), ("l2_policy", -1), ("band_rows", -5), ("struct_size", 4), ("pdl", 2)]:
        bad = _lib.Options()
        L.harris_options_default(ctypes.byref(bad))
        setattr(bad, field, val)
        h = ctypes.c_void_p()
        assert L.harris_init_ex(ctypes.byref(h), 0, ctypes.byref(bad)) == _lib.HARRIS_ERR_INVALID_ARGUMENT
        assert not h.value
    h = ctypes.c_void_p()
    assert L.harris_init_ex(ctypes.byref(h), 0, None) == 0
    L.harris_destroy(h)


def test_band_rows_option_changes_plan_not_bits(cuda_ctx):
    ctx = hb.HarrisContext(0, band_rows=30)
    assert ctx.plan(1076, 1916, batch=4)["band_rows"] == 30
    rgb = torch.from_numpy(synth.synth_numpy(6, 200, 388, seed=5).reshape(2, 3, 200, 388)).cuda()
    assert torch.equal(hb.harris(rgb, ctx=ctx), hb.harris(rgb))


def test_dev_knobs_ignored_without_harris_dev(cuda_ctx, monkeypatch):
    monkeypatch.delenv("HARRIS_DEV", raising=False)
    monkeypatch.setenv("HARRIS_BAND_ROWS", "30")
    monkeypatch.setenv("HARRIS_TMA_CONFIG", "1")
    plain = hb.HarrisContext(0)
    monkeypatch.setenv("HARRIS_DEV", "1")
    dev = hb.HarrisContext(0)
    default = cuda_ctx.plan(1076, 1916, batch=1024)
    assert plain.plan(1076, 1916, batch=1024) == default
    assert default["band_rows"] != 30 and default["tma_config"] != 1
    assert dev.plan(1076, 1916, batch=1024)["band_rows"] == 30
    assert dev.plan(1076, 1916, batch=1024)["tma_config"] == 1


def test_stencil_out_validation(cuda_ctx):
    img = torch.rand(34, 66, device="cuda")
    for bad in [torch.empty(32, 64, device="cuda", dtype=torch.float16),
                torch.empty(32, 64, device="cuda", dtype=torch.bfloat16),
                torch.empty(32, 64, dtype=torch.float32),  # host
                torch.empty(32, 63, device="cuda")]:
        with pytest.raises(ValueError):
            hb.stencil3x3_sep(img, out=bad)


def test_grouping_out_validation(cuda_ctx):
    rgb = torch.from_numpy(synth.synth_numpy(3, 36, 68, seed=3)).cuda()
    for bad in [torch.empty(32, 64, device="cuda", dtype=torch.float16),
                torch.empty(32, 64),
                torch.empty(64, 32, device="cuda").t(),
                torch.empty(32, 60, device="cuda")]:
        with pytest.raises(ValueError):
            hb.harris_grouping(rgb, 1, out=bad)
    ref = hb.harris(rgb, exact=True)
    for g in (1, 2, 3, 4):
        out = torch.empty(32, 64, device="cuda")
        # scratch given as a bf16 buffer of enough BYTES: sized through element_size()
        need = int(_lib.lib().harris_grouping_scratch_bytes(g, 32, 64))
        scratch = torch.empty(max(need // 2, 1), dtype=torch.bfloat16, device="cuda") if need else None
        assert torch.equal(hb.harris_grouping(rgb, g, out=out, scratch=scratch, exact=True), ref)


def test_u8_host_path_honours_out(cuda_ctx):
    rng = np.random.default_rng(4)
    hwc = rng.integers(0, 256, size=(2, 40, 70, 3), dtype=np.uint8)
    out = np.full((2, 36, 66), np.nan, dtype=np.float32)
    ret = hb.harris_u8(hwc, out=out, exact=True)
    assert ret is out
    f32 = np.ascontiguousarray(hwc.transpose(0, 3, 1, 2)).astype(np.float32) / np.float32(255.0)
    for b in range(2):
        assert np.array_equal(out[b], cref.harris_f32(f32[b]))
    with pytest.raises(ValueError):
        hb.harris_u8(hwc, out=np.empty((2, 36, 65), np.float32))
    t = torch.empty(2, 36, 66)
    assert hb.harris_u8(torch.from_numpy(hwc), out=t) is t


def test_host_pipeline_error_returns_after_drain(cuda_ctx):
    """A failing chunk must not return while earlier chunks still read the host buffers:
    a bad flag combination fails inside run() after the first H2D was queued; the call
    returns an error and every stream is idle afterwards."""
    rgb = np.ascontiguousarray(synth.synth_numpy(3, 40, 70, seed=1))
    out = np.empty((36, 66), np.float32)
    L = _lib.lib()
    # FORCE_TMA on a width TMA cannot describe (70 floats: pitch 280 B, not a multiple of 16)
    rc = L.harris_run_host(cuda_ctx.handle, out.ctypes.data, 66, 36, 66, rgb.ctypes.data, 1, 0.04,
                           _lib.FLAG_FORCE_TMA)
    assert rc == _lib.HARRIS_ERR_ALIGNMENT
    # the ctx is still usable
    got = hb.harris(rgb, exact=True)
    assert np.array_equal(np.asarray(got), cref.harris_f32(rgb))


@pytest.mark.parametrize("pdl", [True, "independent"])
def test_pdl_launches_bit_identical_and_stream_ordered(cuda_ctx, pdl):
    plain_ctx = hb.HarrisContext(0, pdl=False)  # harris_options.pdl = 0: plain launches
    """PDL launches (HARRIS_FLAG_PDL / _PDL_INDEPENDENT) give the same bits as plain launches on
    every kernel path, and stream order holds for the work around them: a producer kernel
    (synth_) right before a PDL-waiting launch, and a consumer (clone) right after a chain."""
    shapes = [(70, 260), (70, 262), (72, 263), (71, 263), (1536, 2560)]
    for H, W in shapes:
        x = torch.empty((3, H, W), device="cuda")
        ref_x = torch.from_numpy(synth.synth_numpy(3, H, W, seed=H * W)).cuda()
        plain = hb.harris(ref_x, ctx=plain_ctx)
        for rep in range(3):
            x.zero_()
            torch.cuda.synchronize()
            hb.synth_(x, seed=H * W)             # producer on the stream
            y = hb.harris(x, pdl=True)           # waits for the producer (mode 1)
            z = hb.harris(ref_x, pdl=pdl)        # independent of the previous launch
            yc, zc = y.clone(), z.clone()        # consumers after the chain
            torch.cuda.synchronize()
            assert torch.equal(yc, plain), (H, W, rep)
            assert torch.equal(zc, plain), (H, W, rep)
    img = torch.from_numpy(synth.synth_numpy(1, 40, 132, seed=2)[0]).cuda()
    assert torch.equal(hb.stencil3x3_sep(img, pdl=pdl), hb.stencil3x3_sep(img))
    u8 = torch.randint(0, 256, (40, 70, 3), dtype=torch.uint8, device="cuda")
    assert torch.equal(hb.harris_u8(u8, pdl=pdl), hb.harris_u8(u8))


def test_harris_frames_ring(cuda_ctx):
    """harris_run_frames: a ring of distinct frames, one launch each, chained with PDL; equal
    to one harris() per frame, also when the ring is rewritten by a producer right before the
    call and consumed right after it, and under CUDA-graph replay."""
    H, W, K = 516, 900, 6
    xs = [torch.empty((3, H, W), device="cuda") for _ in range(K)]
    for it in range(3):
        for i, x in enumerate(xs):
            hb.synth_(x, seed=100 * it + i)
        outs = hb.harris_frames(xs)
        copies = [o.clone() for o in outs]
        torch.cuda.synchronize()
        for i, x in enumerate(xs):
            assert torch.equal(copies[i], hb.harris(x)), (it, i)
    # graph capture / replay of the ring
    outs = [torch.empty((H - 4, W - 4), device="cuda") for _ in range(K)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        hb.harris_frames(xs, outs)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            hb.harris_frames(xs, outs)
    for o in outs:
        o.zero_()
    g.replay()
    torch.cuda.synchronize()
    for i, x in enumerate(xs):
        assert torch.equal(outs[i], hb.harris(x)), i
    with pytest.raises(ValueError):
        hb.harris_frames(xs, [outs[0]] * K)  # outputs must be distinct
    vp = ctypes.c_void_p
    L = _lib.lib()
    same = (vp * 2)(outs[0].data_ptr(), outs[0].data_ptr())
    ins = (vp * 2)(xs[0].data_ptr(), xs[1].data_ptr())
    assert L.harris_run_frames(cuda_ctx.handle, same, W - 4, H - 4, W - 4, ins, W, H * W, 2, 0.04, 0,
                               None) == _lib.HARRIS_ERR_INVALID_ARGUMENT  # the C-ABI checks it too


def test_harris_frames_u8_ring(cuda_ctx):
    """harris_run_frames_u8: a ring of interleaved u8 frames, one PDL-chained launch each,
    equal to one harris_u8 call per frame (EXACT and FAST), also with odd widths (bulk rows)."""
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    for H, W in [(300, 516), (131, 517)]:
        xs = [torch.randint(0, 256, (H, W, 3), dtype=torch.uint8, device="cuda", generator=g) for _ in range(5)]
        for exact in (False, True):
            outs = hb.harris_frames(xs, exact=exact)
            torch.cuda.synchronize()
            for i, x in enumerate(xs):
                assert torch.equal(outs[i], hb.harris_u8(x, exact=exact)), (H, W, exact, i)


@pytest.mark.parametrize("band_rows", [0, 7, 30, 136])
def test_u8_fast_bits_do_not_depend_on_the_tile_plan(cuda_ctx, band_rows):
    """The u8 ops sum box rows in pairs; tiles start on even rows, so every tile plan (forced
    heights, the frame-stream plan of PDL-independent frames) gives the same FAST bits."""
    g = torch.Generator(device="cuda")
    g.manual_seed(band_rows)
    ctx = hb.HarrisContext(0, band_rows=band_rows or None)
    for H, W in [(300, 516), (301, 1918), (1080, 1080)]:
        x = torch.randint(0, 256, (2, H, W, 3), dtype=torch.uint8, device="cuda", generator=g)
        ref = hb.harris_u8(x)
        assert torch.equal(hb.harris_u8(x, ctx=ctx), ref), (band_rows, H, W)
        for b in range(2):
            assert torch.equal(hb.harris_u8(x[b], ctx=ctx, pdl="independent"), ref[b]), (band_rows, H, W, b)
