import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2212_12035_b200 as hb
B, H, W = 128, 1080, 1920
x = torch.randint(0, 256, (B, H, W, 3), dtype=torch.uint8, device="cuda")
out = torch.empty((B, H - 4, W - 4), device="cuda")
for _ in range(4):
    hb.harris_u8(x, out=out)
torch.cuda.synchronize()
