"""Dev probe: where do the configs[1] (1536x2560) microseconds go?

Per TMA config (HARRIS_TMA_CONFIG) and band height (HARRIS_BAND_ROWS), the device
time of one launch
  warm   : back to back, input L2-resident (63 MB < 126 MB L2)
  flush  : L2 flushed (1 GiB write + 1 GiB read) before every launch
  primed : flushed, then a tiny launch of the same kernel (same smem carveout) before
           the timed one
python tools/probe_small2.py [cfgs] [band_rows list]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import sys, torch, json
sys.path.insert(0, ROOT)
import paper_2212_12035_b200 as hb
H, W = 1536, 2560
x = torch.empty((3, H, W), device='cuda'); hb.synth_(x, seed=12035)
out = torch.empty((H - 4, W - 4), device='cuda')
xt = torch.empty((3, 12, 136), device='cuda'); hb.synth_(xt, seed=1)
ot = torch.empty((8, 132), device='cuda')
s1 = torch.empty(1 << 28, device='cuda'); s2 = torch.empty(1 << 28, device='cuda')
for _ in range(10): hb.harris(x, out=out)
def timed(pre):
    evs = []
    for _ in range(40):
        pre()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); hb.harris(x, out=out); e1.record(); evs.append((e0, e1))
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in evs)
    return round(ts[len(ts) // 2], 2), round(ts[0], 2)
def flush():
    s1.fill_(0.0); s2.sum()
def primed():
    flush(); hb.harris(xt, out=ot)
r = dict(warm=timed(lambda: None), flush=timed(flush), primed=timed(primed))
p = hb.context().plan(H - 4, W - 4)
r['plan'] = dict(band_rows=p['band_rows'], tiles=p['tiles'], grid=p['grid_ctas'])
print(json.dumps(r))
"""


def main():
    cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "6,0,8").split(",")]
    rows = [int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "0").split(",")]
    for cfg in cfgs:
        for br in rows:
            env = dict(os.environ, HARRIS_DEV="1", HARRIS_TMA_CONFIG=str(cfg))
            if br:
                env["HARRIS_BAND_ROWS"] = str(br)
            r = subprocess.run([sys.executable, "-c", CODE.replace("ROOT", repr(ROOT))], env=env,
                               capture_output=True, text=True)
            print(f"cfg {cfg} band_rows {br or 'auto'}:", r.stdout.strip()[-400:] or r.stderr[-400:], flush=True)


if __name__ == "__main__":
    main()
