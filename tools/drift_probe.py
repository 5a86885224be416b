"""Dev: DRAM read bytes per image vs number of waves (tests the warp-drift theory)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402

B = int(sys.argv[1])
x = torch.empty((B, 3, 1080, 1920), device="cuda")
hb.synth_(x.view(B * 3, 1080, 1920), seed=12035)
out = torch.empty((B, 1076, 1916), device="cuda")
for _ in range(4):
    hb.harris(x, out=out)
torch.cuda.synchronize()
print(hb.context().plan(1076, 1916, B))
