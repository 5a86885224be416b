"""GPU: the fused compute + gather over peer memory (paper_2212_12035_b200/peer.py).

Two processes share the box's one B200 (CUDA IPC works between processes on the same
device exactly as between NVLink peers; a gloo group only exchanges the handles once).
Each rank runs the fused kernel with its output aimed into the root's result buffer
(harris_run_notify) and the root's stream waits on the ranks' flags on the device:
the gathered result must be bit-identical to the whole-image kernel output, every
step, and (exact order) to the C oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)


def _rows_worker(rank, port, H, W, steps, exact, errfile):
    try:
        _init(rank, port)
        import paper_2212_12035_b200 as hb
        from paper_2212_12035_b200 import peer, shard
        from oracle import synth
        n, m = H - 4, W - 4
        rgb = torch.from_numpy(synth.synth_numpy(3, H, W, seed=H + 31 * W)).cuda()
        band = shard.row_bands(n, WORLD)[rank]
        g = peer.PeerGather((n, m), root=0)
        ref = hb.harris(rgb, exact=exact)
        for step in range(steps):
            res = g.run_rows(shard.band_view(rgb, band), band.out_row0, exact=exact)
            if rank == 0:
                got = res.clone()  # stream-ordered after the flag wait
                torch.cuda.synchronize()
                assert torch.equal(got, ref), f"step {step}: max |d| {(got - ref).abs().max().item()}"
                if exact:
                    from oracle import cref
                    assert np.array_equal(got.cpu().numpy(), cref.harris_f32(rgb.cpu().numpy()))
        g.check()
        g.close()
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001 - report to the parent
        with open(errfile, "a") as f:
            f.write(f"rank {rank}: {e!r}\n")
        raise


def _images_worker(rank, port, B, H, W, steps, errfile):
    try:
        _init(rank, port)
        import paper_2212_12035_b200 as hb
        from paper_2212_12035_b200 import peer, shard
        n, m = H - 4, W - 4
        x = torch.empty((B, 3, H, W), dtype=torch.float32, device="cuda")
        hb.synth_(x.view(B * 3, H, W), seed=12035)
        s = shard.image_shards(B, WORLD)[rank]
        g = peer.PeerGather((B, n, m), root=0, buffers=2)
        ref = hb.harris(x)
        for step in range(steps):
            res = g.run_images(x[s.image0: s.image0 + s.images], s.image0)
            if rank == 0:
                assert torch.equal(res, ref), f"step {step}"
        g.check()
        g.close()
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001
        with open(errfile, "a") as f:
            f.write(f"rank {rank}: {e!r}\n")
        raise


def _spawn(fn, args, tmp_path):
    err = str(tmp_path / "err.txt")
    try:
        mp.spawn(fn, args=(_free_port(),) + args + (err,), nprocs=WORLD, join=True)
    except Exception:
        msg = open(err).read() if os.path.exists(err) else ""
        pytest.fail(f"peer gather worker failed:\n{msg}")


@pytest.mark.parametrize("H,W,exact", [(260, 516, False), (133, 132, True), (1028, 2052, False)])
def test_peer_gather_row_bands(tmp_path, H, W, exact):
    _spawn(_rows_worker, (H, W, 4, exact), tmp_path)


def test_peer_gather_ragged_band_generic_width(tmp_path):
    # W % 4 != 0: the generic kernel runs, its completion goes through the signal kernel
    _spawn(_rows_worker, (37, 71, 3, True), tmp_path)


def test_peer_gather_images(tmp_path):
    _spawn(_images_worker, (5, 68, 136, 3), tmp_path)
