"""GPU parity at the bench's full sizes for the other workloads `bench.py` reports
(`extra.batch_u8`, `extra.batch_binomial`, `extra.batch_binomial_window`): every image of the
1024 × 1080×1920 batch, each computed in ONE launch exactly as the bench runs it.

* u8 interleaved ingest: EXACT equals the C f32 oracle on byte/255 bit for bit, FAST meets the
  §8(d) tolerance of the f64 oracle on byte/255.
* separable 3×3 (the reference's binomial goal): EXACT equals the C f32 oracle bit for bit,
  FAST is within 1e-6 (normalised L∞) of the f64 oracle in the reference's separated order.
* Harris with the binomial window: EXACT equals the C f32 window oracle bit for bit, FAST meets
  the §8(d) tolerance of the f64 window oracle (pinned to the reference evaluator).
"""
import numpy as np
import pytest
import torch

from oracle import cref, synth

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_2212_12035_b200")

B, H, W = 1024, 1080, 1920
CHUNK = 64


def test_fullsize_u8_batch(cuda_ctx):
    g = torch.Generator(device="cuda")
    g.manual_seed(12035)
    x8 = torch.randint(0, 256, (B, H, W, 3), dtype=torch.uint8, device="cuda", generator=g)
    ex = hb.harris_u8(x8, exact=True)
    fast = hb.harris_u8(x8)
    torch.cuda.synchronize()
    worst = 0.0
    for b0 in range(0, B, CHUNK):
        hwc = x8[b0:b0 + CHUNK].cpu().numpy()
        planes = np.ascontiguousarray(hwc.transpose(0, 3, 1, 2)).astype(np.float32) / np.float32(255.0)
        e = ex[b0:b0 + CHUNK].cpu().numpy()
        f = fast[b0:b0 + CHUNK].cpu().numpy()
        ref32 = cref.harris_f32_batched(np.ascontiguousarray(planes))
        assert np.array_equal(e, ref32), f"u8 exact: images [{b0}, {b0 + CHUNK})"
        for i in range(planes.shape[0]):
            ok, m = synth.within_tolerance(f[i], cref.harris_f64(planes[i]))
            assert ok, (b0 + i, m)
            worst = max(worst, m["norm_linf"])
    print(f"\nu8 batch FAST vs f64, all {B} images: worst norm L-inf {worst:.3g}")


def test_fullsize_stencil_batch(cuda_ctx):
    x = torch.empty((B, H, W), device="cuda")
    hb.synth_(x, seed=12035)
    ex = hb.stencil3x3_sep(x, exact=True)
    fast = hb.stencil3x3_sep(x)
    torch.cuda.synchronize()
    worst = 0.0
    for b0 in range(0, B, CHUNK):
        host = x[b0:b0 + CHUNK].cpu().numpy()
        e = ex[b0:b0 + CHUNK].cpu().numpy()
        f = fast[b0:b0 + CHUNK].cpu().numpy()
        for i in range(host.shape[0]):
            assert np.array_equal(e[i], cref.sep3x3_f32(host[i])), b0 + i
            ref = cref.sep3x3_f64(host[i], form=1)
            nl = float(np.max(np.abs(f[i] - ref)) / np.max(np.abs(ref)))
            assert nl <= 1e-6, (b0 + i, nl)
            worst = max(worst, nl)
    print(f"\nbinomial stencil batch FAST vs f64, all {B} planes: worst norm L-inf {worst:.3g}")


def test_fullsize_binomial_window_batch(cuda_ctx):
    x = torch.empty((B, 3, H, W), device="cuda")
    hb.synth_(x.view(B * 3, H, W), seed=12035)
    ex = hb.harris(x, exact=True, window="binomial")
    fast = hb.harris(x, window="binomial")
    torch.cuda.synchronize()
    worst = 0.0
    for b0 in range(0, B, CHUNK):
        host = x[b0:b0 + CHUNK].cpu().numpy()
        e = ex[b0:b0 + CHUNK].cpu().numpy()
        f = fast[b0:b0 + CHUNK].cpu().numpy()
        for i in range(host.shape[0]):
            assert np.array_equal(e[i], cref.harris_f32(host[i], window="binomial")), b0 + i
            ok, m = synth.within_tolerance(f[i], cref.harris_f64(host[i], window="binomial"))
            assert ok, (b0 + i, m)
            worst = max(worst, m["norm_linf"])
    print(f"\nbinomial-window batch FAST vs f64, all {B} images: worst norm L-inf {worst:.3g}")
