"""A/B timing of one shape: python tools/perf_shape.py {f32,f32crop,f32win,u8,sep,seppad,sepcrop} B H W [reps]; HARRIS_LIB selects the .so."""
import sys, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2212_12035_b200 as hb
kind, B, H, W = sys.argv[1], *map(int, sys.argv[2:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 10
g = torch.Generator(device="cuda"); g.manual_seed(12035)
if kind == "u8":
    x = torch.randint(0, 256, (B, H, W, 3), dtype=torch.uint8, device="cuda", generator=g)
    f = lambda: hb.harris_u8(x, out=out)
elif kind == "sep":
    x = torch.rand((B, H, W), device="cuda", generator=g)
    out2 = torch.empty((B, H - 2, W - 2), device="cuda")
    f = lambda: hb.stencil3x3_sep(x, out=out2)
elif kind == "seppad":  # thesis-style output pitch = input width (16-byte aligned rows)
    x = torch.rand((B, H, W), device="cuda", generator=g)
    out2 = torch.empty((B, H - 2, W), device="cuda")[..., :W - 2]
    f = lambda: hb.stencil3x3_sep(x, out=out2)
elif kind == "sepcrop":  # column-crop view x[..., :W] of (W+2)-pitch planes: TMA loads, m = W - 2
    x = torch.rand((B, H, W + 2), device="cuda", generator=g)[..., :W]
    out2 = torch.empty((B, H - 2, W - 2), device="cuda")
    f = lambda: hb.stencil3x3_sep(x, out=out2)
elif kind == "f32crop":  # column-crop view: base 4-byte aligned only
    x = torch.rand((B, 3, H, W + 1), device="cuda", generator=g)[..., 1:]
    f = lambda: hb.harris(x, out=out)
elif kind == "f32win":  # Harris with the binomial window
    x = torch.rand((B, 3, H, W), device="cuda", generator=g)
    f = lambda: hb.harris(x, out=out, window="binomial")
else:
    x = torch.rand((B, 3, H, W), device="cuda", generator=g)
    f = lambda: hb.harris(x, out=out)
out = torch.empty((B, H - 4, W - 4), device="cuda")
for _ in range(3): f()
torch.cuda.synchronize()
evs = []
for _ in range(reps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); f(); e1.record(); evs.append((e0, e1))
torch.cuda.synchronize()
ts = sorted(a.elapsed_time(b) for a, b in evs)
med = ts[len(ts) // 2]
px = B * (H - 2) * (W - 2) if kind.startswith("sep") else B * (H - 4) * (W - 4)
print(f"{sys.argv[1:]} {'old' if 'HARRIS_LIB' in __import__('os').environ else 'new'} median_ms {med:.4f} MP/s {px/med/1e3:.0f}")
