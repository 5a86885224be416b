"""GPU parity at BASELINE.json's full sizes (configs[1]..configs[4]).

The C oracle (oracle/harris_oracle.c, OpenMP) is fast enough to check every output
pixel of every config: the EXACT-order kernel must equal the C f32 restatement
bit-for-bit over the whole 8192^2 image, the whole 32768^2 image and all 1024 images
of the batch, each computed in ONE launch exactly as the bench runs it.  The shipped
FAST order is checked against the f64 oracle (pinned to the reference evaluator) on
every pixel of every config too — every image of the 1024-image batch and every row of
32768^2 (SURVEY.md §8(d) tolerance, per image; row bands of one image accumulate into one
verdict through synth.ToleranceAccumulator, exactly equal to the whole-image check).  Size-independent properties at full size: the 8 row
bands of 32768^2 (the multi-GPU decomposition, 4-row halo views) reproduce the
single-launch output bit-for-bit.

Inputs come from the device generator (bit-identical to the host one,
test_gpu_parity.py::test_synth_device_matches_host) and are copied back for the
oracle in bounded chunks.
"""
import numpy as np
import pytest
import torch

from oracle import cref, synth

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_2212_12035_b200")
from paper_2212_12035_b200 import shard  # noqa: E402

SEED = 12035


def _image(H, W, seed=SEED):
    x = torch.empty((3, H, W), dtype=torch.float32, device="cuda")
    hb.synth_(x, seed=seed)
    return x


def _check_exact(got: torch.Tensor, rgb_host: np.ndarray, what: str):
    ref = cref.harris_f32(rgb_host)
    g = got.cpu().numpy()
    if not np.array_equal(g, ref):
        bad = np.argwhere(g != ref)
        raise AssertionError(f"{what}: {len(bad)} pixels differ, first at {bad[0].tolist()}")


# thesis evaluation sizes (1536x2560 and 4256x2832, both
# orientations) and the bandwidth-roofline config
# (8190, 8190): row starts not 16-byte aligned -> the cp.async strip engine (K2)
@pytest.mark.parametrize("H,W", [(1536, 2560), (2560, 1536), (4256, 2832), (2832, 4256), (8192, 8192),
                                 (8190, 8190)])
def test_fullsize_single_image(cuda_ctx, H, W):
    x = _image(H, W)
    ex = hb.harris(x, exact=True)
    fast = hb.harris(x)
    torch.cuda.synchronize()
    host = x.cpu().numpy()
    _check_exact(ex, host, f"{H}x{W} exact")
    ok, m = synth.within_tolerance(fast.cpu().numpy(), cref.harris_f64(host))
    assert ok, (H, W, m)


def test_fullsize_batch_1024(cuda_ctx):
    B, H, W = 1024, 1080, 1920
    x = torch.empty((B, 3, H, W), dtype=torch.float32, device="cuda")
    hb.synth_(x.view(B * 3, H, W), seed=SEED)
    ex = hb.harris(x, exact=True)          # one launch over the whole batch (bench config)
    torch.cuda.synchronize()
    for b0 in range(0, B, 64):             # every image, bit-for-bit
        host = x[b0: b0 + 64].cpu().numpy()
        ref = cref.harris_f32_batched(host)
        got = ex[b0: b0 + 64].cpu().numpy()
        assert np.array_equal(got, ref), f"batch exact: images [{b0}, {b0 + 64}) differ"
    del ex
    fast = hb.harris(x)
    torch.cuda.synchronize()
    # every image of the shipped order vs the f64 oracle, per-image tolerance
    worst = {"norm_linf": 0.0, "psnr_db": float("inf")}
    for b0 in range(0, B, 64):
        host = x[b0: b0 + 64].cpu().numpy()
        got = fast[b0: b0 + 64].cpu().numpy()
        for i in range(host.shape[0]):
            ok, m = synth.within_tolerance(got[i], cref.harris_f64(host[i]))
            assert ok, (b0 + i, m)
            worst["norm_linf"] = max(worst["norm_linf"], m["norm_linf"])
            worst["psnr_db"] = min(worst["psnr_db"], m["psnr_db"])
    print(f"\nconfigs[4] FAST vs f64, all {B} images: worst {worst}")


def test_fullsize_image32768_and_row_bands(cuda_ctx):
    H = W = 32768
    n, m = H - 4, W - 4
    free, _ = torch.cuda.mem_get_info()
    if free < (12 + 4 + 4 + 2) << 30:
        pytest.skip("needs ~22 GiB of free device memory")
    x = _image(H, W)
    ex = hb.harris(x, exact=True)
    torch.cuda.synchronize()
    step = 2048
    for r0 in range(0, n, step):             # every output row, bit-for-bit
        rows = min(step, n - r0)
        host = x[:, r0: r0 + rows + 4].cpu().numpy()
        _check_exact(ex[r0: r0 + rows], host, f"32768^2 exact rows [{r0}, {r0 + rows})")
    del ex
    fast = hb.harris(x)
    # the 8-GPU decomposition: each band is a 4-row-halo view of the same image
    parts = [hb.harris(shard.band_view(x, b)) for b in shard.row_bands(n, 8)]
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts, 0), fast), "row bands differ from the single launch"
    del parts
    acc = synth.ToleranceAccumulator()       # every output row vs the f64 oracle, one verdict
    for r0 in range(0, n, step):
        rows = min(step, n - r0)
        host = x[:, r0: r0 + rows + 4].cpu().numpy()
        acc.add(fast[r0: r0 + rows].cpu().numpy(), cref.harris_f64(host))
    ok, mt = acc.result()
    assert ok and mt["pixels"] == n * m, mt
    print(f"\nconfigs[3] FAST vs f64, all {n} rows: {mt}")
