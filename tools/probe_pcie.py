"""Dev: raw pinned PCIe bandwidth with 1..4 concurrent H2D streams, and H2D with a
concurrent D2H of 1/3 the bytes (the e2e traffic mix: 12 B/px in, 4 B/px out)."""
import torch

GB = 1 << 30
h = torch.empty(4 * GB // 4, dtype=torch.float32, pin_memory=True)
d = torch.empty(4 * GB // 4, dtype=torch.float32, device="cuda")
ho = torch.empty(GB // 4 * 4 // 3, dtype=torch.float32, pin_memory=True)
do = torch.empty(GB // 4 * 4 // 3, dtype=torch.float32, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(nstreams, with_d2h=False, reps=3):
    n = h.numel()
    chunk = n // nstreams
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for k in range(nstreams):
            streams[k].wait_event(e0)
            with torch.cuda.stream(streams[k]):
                d[k * chunk:(k + 1) * chunk].copy_(h[k * chunk:(k + 1) * chunk], non_blocking=True)
        if with_d2h:
            with torch.cuda.stream(streams[3]):
                ho.copy_(do, non_blocking=True)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    return round(reps * nstreams * chunk * 4 / t / 1e9, 1), round(reps * ho.numel() * 4 / t / 1e9, 1) if with_d2h else 0


for ns in (1, 2, 3):
    print("H2D streams", ns, "GB/s", run(ns))
print("H2D 1 stream + concurrent D2H (1/3 bytes): H2D, D2H GB/s", run(1, True))
print("H2D 2 streams + concurrent D2H (1/3 bytes): H2D, D2H GB/s", run(2, True))
