import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2212_12035_b200 as hb
H, W, K = 1536, 2560, 9
xs = [torch.rand(3, H, W, device="cuda") for _ in range(K)]
outs = [torch.empty(H - 4, W - 4, device="cuda") for _ in range(K)]
plain = hb.HarrisContext(0, pdl=False)
res = {}
for name, kw in (("graph_plain", dict(ctx=plain)), ("graph_pdlwait", dict(pdl=True)), ("graph_indep", dict(pdl="independent"))):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for x, o in zip(xs, outs): hb.harris(x, out=o, **kw)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for x, o in zip(xs, outs): hb.harris(x, out=o, **kw)
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): g.replay()
    e1.record(); torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) * 1e3 / (20 * K)
    # single graph containing 20 rings back to back
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g2, stream=s):
            for _ in range(20):
                for x, o in zip(xs, outs): hb.harris(x, out=o, **kw)
    g2.replay(); torch.cuda.synchronize()
    e0.record(); g2.replay(); e1.record(); torch.cuda.synchronize()
    res[name + "_1graph180"] = e0.elapsed_time(e1) * 1e3 / (20 * K)
print(json.dumps(res, indent=1))
