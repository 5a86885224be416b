"""GPU: the bench's N>1 code path on a one-GPU box.

Two torchrun ranks share cuda:0 (HARRIS_BENCH_SHARE_GPU=1, gloo for the host-side
collectives — NCCL refuses two ranks on one device): the row-band workload with the fused
peer gather and the image-sharded batch workload (strong scaling by default: the literal
configs[4] batch split over the ranks; weak as a flag) must each print exactly one JSON
line with n_gpus = N.  The numbers themselves are meaningless here (two
processes time-slice one GPU); this checks the plumbing the 8-GPU scaling run uses.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _torchrun(args, timeout=600, nproc=2):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus",
           str(nproc), "--dist-backend", "gloo"] + args
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout,
                       env=dict(os.environ, HARRIS_BENCH_SHARE_GPU="1"))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    return lines[0]


def test_two_rank_row_bands_with_fused_gather():
    d = _torchrun(["--workload", "image8192", "--steps", "3", "--warmup", "3", "--no-e2e", "--gather", "peer"])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["gather"].startswith("fused")
    assert d["gpu_launches"] == 3 * 3


def test_two_rank_weak_scaling_batch():
    d = _torchrun(["--scaling", "weak", "--steps", "3", "--warmup", "3", "--e2e-images", "8", "--e2e-steps", "1"])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["config"]["images"] == 2048 and d["config"]["images_per_gpu"] == 1024
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0


@pytest.mark.parametrize("nproc", [2, 4, 8])
def test_default_batch_line_is_the_literal_config(nproc):
    """The default N>1 batch line (what the driver's scaling run prints) is BASELINE
    configs[4] itself: ONE 1024-image batch of 1920x1080 split over the ranks (strong
    scaling), value = all 1024 images' output pixels / max-over-ranks time."""
    d = _torchrun(["--steps", "2", "--warmup", "3", "--e2e-images", "4", "--e2e-steps", "1"], nproc=nproc,
                  timeout=900)
    c = d["config"]
    assert d["n_gpus"] == nproc and d["scaling"] == "strong"
    assert "configs[4]" in c["workload"] and c["images"] == 1024 and c["images_per_gpu"] == 1024 // nproc
    assert c["output"] == [1024, 1076, 1916] and c["height"] == 1080 and c["width"] == 1920
    px = 1024 * 1076 * 1916
    assert d["value"] == pytest.approx(px * d["steps"] / (d["ms_per_step"] * d["steps"] * 1e-3) / 1e6, rel=1e-9)
    assert d["roofline"]["algorithmic_bytes_per_launch"] == (1024 // nproc) * (12 * 1080 * 1920 + 4 * 1076 * 1916)


def test_four_rank_row_bands_fused_gather():
    """4 ranks, 4 row bands of 8192^2, every band's kernel storing into rank 0's buffer."""
    d = _torchrun(["--workload", "image8192", "--steps", "2", "--warmup", "3", "--no-e2e", "--gather", "peer"],
                  nproc=4)
    assert d["n_gpus"] == 4 and d["value"] > 0 and d["config"]["gather"].startswith("fused")


def test_eight_rank_row_bands_fused_gather():
    """The N = 8 decomposition of the scaling run (8 row bands, 8 peer mappings of rank 0's
    buffer, 8 completion flags), as 8 processes on the one GPU."""
    d = _torchrun(["--workload", "image8192", "--steps", "2", "--warmup", "3", "--no-e2e", "--gather", "peer"],
                  nproc=8, timeout=900)
    assert d["n_gpus"] == 8 and d["value"] > 0 and d["config"]["gather"].startswith("fused")
