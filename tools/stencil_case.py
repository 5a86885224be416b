"""Dev: binomial stencil launches on 128 x 1080x1920 planes for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402

B, H, W = 128, 1080, 1920
x = torch.empty((B, H, W), device="cuda")
hb.synth_(x, seed=12035)
out = torch.empty((B, H - 2, W - 2), device="cuda")
for _ in range(5):
    hb.stencil3x3_sep(x, out=out)
torch.cuda.synchronize()
