"""Dev: a few u8-ingest launches on 128 x 1080x1920 for ncu (-k regex:strip_kernel -s 3 -c 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402

B, H, W = 128, 1080, 1920
g = torch.Generator(device="cuda")
g.manual_seed(12035)
x = torch.randint(0, 256, (B, H, W, 3), dtype=torch.uint8, device="cuda", generator=g)
out = torch.empty((B, H - 4, W - 4), device="cuda")
for _ in range(5):
    hb.harris_u8(x, out=out)
torch.cuda.synchronize()
