"""GPU: seeded random layouts through every kernel path, bit-exact against the oracle.

Each case draws an image size (5..~700 rows/cols), a batch, a row pitch padding, a
channel-plane gap, a base offset (in elements / bytes) and an output pitch, so the
calls land on the TMA path (16-byte aligned layouts), the cp.async K2 path (anything
else) or — with force_generic — K0.  In EXACT order every one of them must equal the C
f32 oracle bit-for-bit; the default order must meet the SURVEY.md §8(d) tolerance.
"""
import numpy as np
import pytest
import torch

from oracle import cref, synth

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_2212_12035_b200")
from paper_2212_12035_b200 import _lib  # noqa: E402

N_CASES = 60


def _case(rng):
    H = int(rng.integers(5, 400))
    W = int(rng.integers(5, 700))
    B = int(rng.choice([1, 1, 2, 3]))
    pad = int(rng.choice([0, 0, 1, 3, 4, 7]))          # extra elements per row
    gap = int(rng.choice([0, 0, 5, 16]))                # extra elements between channel planes
    off = int(rng.choice([0, 0, 1, 2, 4]))              # base offset in elements
    opad = int(rng.choice([0, 0, 1, 4]))                # output row padding
    generic = bool(rng.random() < 0.15)
    return H, W, B, pad, gap, off, opad, generic


@pytest.mark.parametrize("seed", range(N_CASES))
def test_fuzz_f32_layouts(cuda_ctx, seed):
    rng = np.random.default_rng(1000 + seed)
    H, W, B, pad, gap, off, opad, generic = _case(rng)
    pitch = W + pad
    chan = H * pitch + gap
    img_stride = 3 * chan + int(rng.choice([0, 8]))
    rgb = synth.synth_numpy(3 * B, H, W, seed=seed).reshape(B, 3, H, W)
    buf = torch.zeros(off + B * img_stride + 16, device="cuda")
    x = torch.as_strided(buf, (B, 3, H, W), (img_stride, chan, pitch, 1), off)
    x.copy_(torch.from_numpy(rgb))
    n, m = H - 4, W - 4
    obuf = torch.full((B * n * (m + opad) + 8,), -3.0, device="cuda")
    out = torch.as_strided(obuf, (B, n, m), (n * (m + opad), m + opad, 1), 0)
    hb.harris(x, out=out, exact=True, force_generic=generic)
    path = cuda_ctx.last_path
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    for b in range(B):
        assert np.array_equal(got[b], cref.harris_f32(rgb[b])), (seed, H, W, B, pad, gap, off, opad, generic, path, b)
    aligned = off % 4 == 0 and pitch % 4 == 0 and chan % 4 == 0 and (B == 1 or img_stride % 4 == 0)
    k = 2 if pitch % 4 == 2 else 4 if pitch % 2 else 0
    grouped = bool(k) and off % 4 == 0 and chan % 4 == 0 and H % k == 0 and (B == 1 or img_stride % 4 == 0)
    assert path == (_lib.PATH_GENERIC if generic else _lib.PATH_TMA if aligned else
                    (_lib.PATH_PAIR if k == 2 else _lib.PATH_QUAD) if grouped else _lib.PATH_LDG)
    # padding columns of the output were never written
    if opad:
        assert torch.all(obuf[: B * n * (m + opad)].view(B, n, m + opad)[:, :, m:] == -3.0)
    fast = hb.harris(x)
    torch.cuda.synchronize()
    for b in range(B):
        ok, mt = synth.within_tolerance(fast[b].cpu().numpy(), cref.harris_f64(rgb[b]))
        assert ok, (seed, b, mt)
    # every third layout also through the binomial-window variant and a PDL launch (round 2):
    # EXACT bit-exact with the window oracle on whichever kernel the layout selects
    if seed % 3 == 0:
        obuf.fill_(-3.0)
        hb.harris(x, out=out, exact=True, window="binomial", pdl=True)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        for b in range(B):
            assert np.array_equal(got[b], cref.harris_f32(rgb[b], window="binomial")), (seed, b, "window")
        if opad:
            assert torch.all(obuf[: B * n * (m + opad)].view(B, n, m + opad)[:, :, m:] == -3.0)


@pytest.mark.parametrize("seed", range(N_CASES // 2))
def test_fuzz_u8_layouts(cuda_ctx, seed):
    rng = np.random.default_rng(5000 + seed)
    H = int(rng.integers(5, 300))
    W = int(rng.integers(5, 600))
    B = int(rng.choice([1, 2]))
    pad = int(rng.choice([0, 0, 1, 5, 16]))   # bytes per row
    off = int(rng.choice([0, 0, 1, 3, 16]))   # base offset in bytes
    pitch = 3 * W + pad
    img_stride = H * pitch + int(rng.choice([0, 3]))
    planes = synth.synth_numpy(3 * B, H, W, seed=seed, dist=1)
    u8 = np.rint(planes * 255.0).astype(np.uint8).reshape(B, 3, H, W)
    hwc = np.ascontiguousarray(u8.transpose(0, 2, 3, 1))
    f32 = (u8.astype(np.float32) / np.float32(255.0)).astype(np.float32)
    buf = torch.zeros(off + B * img_stride + 16, dtype=torch.uint8, device="cuda")
    x = torch.as_strided(buf, (B, H, W, 3), (img_stride, pitch, 3, 1), off)
    x.copy_(torch.from_numpy(hwc))
    got = hb.harris_u8(x, exact=True)
    path = cuda_ctx.last_path
    torch.cuda.synchronize()
    for b in range(B):
        assert np.array_equal(got[b].cpu().numpy(), cref.harris_f32(f32[b])), (seed, H, W, B, pad, off, path, b)
    base_ok = off % 16 == 0 and (B == 1 or img_stride % 16 == 0)
    k = 2 if pitch % 16 == 8 else 4 if pitch % 8 == 4 else 0
    expect = (_lib.PATH_TMA if base_ok and pitch % 16 == 0 else
              (_lib.PATH_PAIR if k == 2 else _lib.PATH_QUAD) if base_ok and k and H % k == 0 else _lib.PATH_LDG)
    assert path == expect, (seed, H, W, B, pad, off, path)
