"""Launch-to-launch variance of the fused kernel on the batch workload (dev tool).

Prints per-launch CUDA-event times of N back-to-back launches and NVML samples
(SM/memory clock, power, temperature, clock-event reasons) taken during them.
"""
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_2212_12035_b200 as hb  # noqa: E402


def main():
    n_launch = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    B, H, W = 1024, 1080, 1920
    x = torch.empty((B, 3, H, W), device="cuda")
    hb.synth_(x.view(B * 3, H, W), seed=12035)
    out = torch.empty((B, H - 4, W - 4), device="cuda")
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    limits = {}
    for name, fn in (("enforced_w", "nvmlDeviceGetEnforcedPowerLimit"), ("mgmt_limit_w", "nvmlDeviceGetPowerManagementLimit"),
                     ("default_w", "nvmlDeviceGetPowerManagementDefaultLimit")):
        try:
            limits[name] = getattr(pynvml, fn)(h) / 1000.0
        except Exception as e:  # pragma: no cover
            limits[name] = repr(e)
    mode = os.environ.get("VARIANCE_MODE", "harris")
    samples = []
    stop = threading.Event()

    def loop():
        while not stop.is_set():
            try:
                samples.append(dict(
                    t=time.perf_counter(),
                    sm=pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                    mem=pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                    pw=pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                    temp=pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU),
                    rsn=pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            time.sleep(0.002)

    flat = x.view(-1)
    half = flat.numel() // 2

    def launch():
        if mode == "copy":   # plain device copy of the same byte volume (read 25.5 GB, write 8.4 GB)
            out.view(-1).copy_(flat[: out.numel()])
            flat[out.numel(): out.numel() * 2].copy_(flat[2 * out.numel(): 3 * out.numel()])
        else:
            hb.harris(x, out=out)

    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    th = threading.Thread(target=loop, daemon=True)
    th.start()
    evs = []
    t0 = time.perf_counter()
    for _ in range(n_launch):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        launch()
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    stop.set()
    th.join()
    ts = [a.elapsed_time(b) for a, b in evs]
    inside = [s for s in samples if t0 <= s["t"] <= t1]
    print(json.dumps({"ms": [round(t, 4) for t in ts],
                      "sm_mhz": sorted({s["sm"] for s in inside}), "mem_mhz": sorted({s["mem"] for s in inside}),
                      "power_w": [round(min(s["pw"] for s in inside)), round(max(s["pw"] for s in inside))],
                      "temp_c": [min(s["temp"] for s in inside), max(s["temp"] for s in inside)],
                      "reasons_or": hex(sum({s["rsn"] for s in inside})), "samples": len(inside),
                      "limits": limits, "mode": mode}))


if __name__ == "__main__":
    main()
