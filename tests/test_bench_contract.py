"""CPU: the bench.py contract the driver depends on.

* `--impl reference` (the reference's CPU path, oracle port) prints ONE JSON line with
  the metric / unit / config of the GPU arm plus `impl`, `cpu_baseline`, `e2e`;
* under torchrun with 2 ranks only rank 0 prints it and every rank exits 0;
* the GPU arm fails loudly without a GPU (no CPU fallback behind the product path);
* the bench's own accounting helpers (workload shards, algorithmic bytes).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")
sys.path.insert(0, ROOT)


def _run(args, timeout=300, env=None):
    return subprocess.run([sys.executable] + args, cwd=ROOT, capture_output=True, text=True, timeout=timeout,
                          env=dict(os.environ, **(env or {})))


def _json_lines(out: str):
    return [json.loads(line) for line in out.splitlines() if line.startswith("{")]


def test_reference_arm_line():
    r = _run([BENCH, "--impl", "reference", "--steps", "2", "--warmup", "3", "--ref-images", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    baseline = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["metric"] == baseline["metric"]
    assert d["impl"] == "reference" and d["unit"] == "MP/s" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "configs[4]" in d["config"]["workload"]
    # both thesis CPU schedules are timed; the arm runs the faster one
    v = cb["variants"]
    assert v["cbuf"]["value"] > 0 and v["rrot"]["value"] > 0 and cb["variant"] in ("cbuf", "rrot")
    assert v["rrot_over_cbuf"] == pytest.approx(v["rrot"]["value"] / v["cbuf"]["value"])
    assert d["config"]["same_as_gpu_arm"] is False  # --ref-images 1: a prefix of the batch


def test_reference_workload_is_the_whole_batch_by_default(monkeypatch):
    """Without --ref-images the reference arm's per-step input is every image of the
    workload (same config as the GPU arm), regenerated bit-exactly on the host."""
    import bench
    from oracle import synth
    wl = dict(bench.WORKLOADS["batch"], B=5, H=40, W=70)
    x, px, desc, same = bench.reference_workload(wl, None)
    assert same and x.shape == (5, 3, 40, 70) and px == 5 * 36 * 66 and "all 5" in desc
    assert np.array_equal(x.reshape(15, 40, 70), synth.synth_numpy(15, 40, 70, seed=bench.SEED))
    monkeypatch.setattr(bench, "host_mem_available", lambda: 2 * 3 * (12 * 40 * 70 + 4 * 36 * 66))
    x, _, desc, same = bench.reference_workload(wl, None)
    assert not same and x.shape[0] == 3 and "first 3 of 5" in desc


def test_reference_arm_under_torchrun_prints_once():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = _run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
              "--master-port", str(port), BENCH, "--impl", "reference", "--gpus", "2", "--steps", "1",
              "--warmup", "3", "--ref-images", "1"], timeout=400)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"


def test_gpu_arm_fails_loudly_without_a_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = _run([BENCH, "--steps", "1", "--warmup", "3", "--no-e2e", "--no-extra", "--no-cpu-baseline"], timeout=200)
    assert r.returncode != 0
    assert not _json_lines(r.stdout)


def test_workload_accounting():
    import bench
    wl = bench.WORKLOADS["batch"]
    sh = bench.Shard(wl, world=1, rank=0)
    assert sh.total_px == 1024 * 1076 * 1916 == sh.local_px
    assert sh.algorithmic_bytes() == 1024 * (12 * 1080 * 1920 + 4 * 1076 * 1916)
    # weak scaling: every rank owns a full 1024-image batch, global images disjoint
    shards = [bench.Shard(wl, world=8, rank=r, scaling="weak") for r in range(8)]
    assert [s.b0 for s in shards] == [r * 1024 for r in range(8)]
    assert all(s.nb == 1024 for s in shards) and shards[0].total_px == 8 * 1024 * 1076 * 1916
    # strong scaling: one batch split, row bands: one image split with a 4-row halo each
    strong = [bench.Shard(wl, world=8, rank=r, scaling="strong") for r in range(8)]
    assert sum(s.nb for s in strong) == 1024
    img = bench.WORKLOADS["image32768"]
    bands = [bench.Shard(img, world=8, rank=r) for r in range(8)]
    assert sum(b.rows for b in bands) == 32764
    assert all(b.in_rows == b.rows + 4 for b in bands)
    assert sum(b.algorithmic_bytes() for b in bands) == sum(12 * (b.rows + 4) * 32768 + 4 * b.rows * 32764
                                                             for b in bands)


def test_clock_summary_reasons():
    import bench
    cs = bench.ClockSampler.__new__(bench.ClockSampler)
    cs.ok, cs.sm_max = True, 1965
    cs.samples = [(0.0, 1965, 0x0), (1.0, 1900, 0x4), (2.0, 1965, 0x1), (9.0, 1000, 0x40)]
    s = cs.summary(0.5, 2.5)
    assert s["sm_mhz"] == pytest.approx((1900 + 1965) / 2) and s["samples"] == 2
    assert s["reasons"] == ["sw_power_cap"]  # gpu_idle is not a throttle reason
