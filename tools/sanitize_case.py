"""Dev: one small launch of every kernel path, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Prints the paths it exercised."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402
from paper_2212_12035_b200 import _lib  # noqa: E402

ctx = hb.context(0)
seen = []


def f32(B, H, W, off=0, **kw):
    buf = torch.rand(off + B * 3 * H * W, device="cuda")
    x = buf[off:].view(B, 3, H, W)
    for exact in (False, True):
        hb.harris(x if B > 1 else x[0], exact=exact, **kw)
        seen.append(("f32", B, H, W, off, exact, ctx.last_path, kw.get("force_generic", False)))


def u8(B, H, W, off=0, **kw):
    buf = torch.randint(0, 256, (off + B * H * W * 3,), dtype=torch.uint8, device="cuda")
    x = buf[off:].view(B, H, W, 3)
    for exact in (False, True):
        hb.harris_u8(x if B > 1 else x[0], exact=exact, **kw)
        seen.append(("u8", B, H, W, off, exact, ctx.last_path))


f32(1, 70, 264)            # TMA, short tiles -> scalar core
f32(1, 300, 1028)          # TMA dual-strip core
f32(3, 41, 388)            # TMA dual, strip pairs straddling images
f32(2, 37, 71)             # K1b bulk rows (width % 4 != 0, height % 4 != 0)
f32(1, 40, 136, off=1)     # K1b (4-byte aligned base)
f32(2, 38, 262)            # K1p pair-row TMA (pitch = 2 mod 4, even height)
f32(2, 40, 263)            # K1q quad-row TMA (odd pitch, height % 4 == 0)
f32(1, 37, 71, force_generic=True)  # K0
u8(2, 40, 400)             # u8 TMA
u8(2, 37, 263, off=1)      # u8 K1b bulk rows
u8(1, 29, 131, off=15)     # u8 K1b, ragged last strip, base 15 bytes past alignment
img = torch.rand(2, 50, 260, device="cuda")
hb.stencil3x3_sep(img)
hb.stencil3x3_sep(img, exact=True)
for off in (1, 3):         # stencil K1b bulk rows (unaligned base, odd pitch)
    buf = torch.rand(off + 2 * 50 * 263, device="cuda")
    hb.stencil3x3_sep(buf[off:].view(2, 50, 263))
    hb.stencil3x3_sep(buf[off:].view(2, 50, 263), exact=True)
for g in (1, 2, 3, 4):
    for exact in (False, True):  # FAST: strip-engine groupings (round 2); EXACT: Appendix-B kernels
        hb.harris_grouping(torch.rand(3, 40, 132, device="cuda"), g, exact=exact)
# round 2: stencil TMA-store epilogue (config 3 on a column-crop view with a 16-byte aligned
# output pitch), realigned stores (contiguous 1918-wide-style outputs), binomial window
# (TMA configs 0 / 6 and generic), PDL launches, the frames API
dev_ctx = None
os.environ["HARRIS_DEV"] = "1"
os.environ["HARRIS_SEP_CONFIG"] = "3"
ts_ctx = hb.HarrisContext(0)
del os.environ["HARRIS_SEP_CONFIG"], os.environ["HARRIS_DEV"]
planes = torch.rand(2, 40, 134, device="cuda")
hb.stencil3x3_sep(planes[..., :130], ctx=ts_ctx, out=torch.empty(2, 38, 132, device="cuda")[..., :128])
hb.stencil3x3_sep(torch.rand(2, 41, 132, device="cuda"))          # m = 130: realigned 16-byte stores
for kw in ({}, {"exact": True}, {"force_generic": True}):
    hb.harris(torch.rand(3, 70, 264, device="cuda"), window="binomial", **kw)
    hb.harris(torch.rand(3, 300, 1028, device="cuda"), window="binomial", **kw)
x0 = torch.rand(3, 70, 264, device="cuda")
hb.harris(x0, pdl=True)
hb.harris(x0, pdl="independent")
hb.harris_frames([torch.rand(3, 64, 260, device="cuda") for _ in range(3)])
x = torch.rand(3, 40, 136, device="cuda")
out = torch.empty(36, 132, device="cuda")
flag = torch.zeros(2, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
L = _lib.lib()
assert L.harris_run_notify(ctx.handle, out.data_ptr(), 132, 36 * 132, 36, 132, x.data_ptr(), 136, 40 * 136,
                           3 * 40 * 136, 1, 0.04, 0, flag.data_ptr(), 1, st) == 0
assert L.harris_peer_wait(flag.data_ptr(), 1, 1, flag.data_ptr() + 4, 1_000_000_000, st) == 0
torch.cuda.synchronize()
assert int(flag[0].item()) == 1 and int(flag[1].item()) == 0
paths = sorted({s[-2] if s[0] == "f32" else s[-1] for s in seen})
print("ok; paths exercised:", paths, "cases:", len(seen))
