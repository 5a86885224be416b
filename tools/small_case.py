"""Dev: a few configs[1] (1536x2560) launches for ncu (-k regex:strip_kernel -s 5 -c 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402

H, W = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (1536, 2560)))
x = torch.empty((3, H, W), device="cuda")
hb.synth_(x, seed=12035)
out = torch.empty((H - 4, W - 4), device="cuda")
for _ in range(8):
    hb.harris(x, out=out)
torch.cuda.synchronize()
print(hb.context().plan(H - 4, W - 4))
