"""Dev: unaligned-width (K2) launches on 8190x8190 for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402

H = W = 8190
x = torch.empty((3, H, W), device="cuda")
hb.synth_(x, seed=1)
out = torch.empty((H - 4, W - 4), device="cuda")
for _ in range(5):
    hb.harris(x, out=out)
torch.cuda.synchronize()
