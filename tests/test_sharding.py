"""CPU: multi-GPU partitioning logic (row bands with a 4-row halo, image shards,
gather to root) on a world_size-2 gloo group.  Each rank computes its shard with
the C oracle standing in for the device kernel (test infrastructure); the
gathered result must be bit-identical to the whole-image oracle output, which is
exactly the property the fused kernel has on the GPU (test_gpu_parity.py
test_row_band_views_bitexact)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2212_12035_b200 import shard


def test_row_bands_cover_and_balance():
    for n in (1, 2, 7, 100, 32764):
        for G in (1, 2, 3, 4, 8):
            bands = shard.row_bands(n, G)
            assert sum(b.out_rows for b in bands) == n
            assert bands[0].out_row0 == 0
            for a, b in zip(bands, bands[1:]):
                assert a.out_row0 + a.out_rows == b.out_row0
            sizes = [b.out_rows for b in bands]
            assert max(sizes) - min(sizes) <= 1
            for b in bands:
                assert b.in_rows == (b.out_rows + 4 if b.out_rows else 0)


def test_config4_band_geometry():
    # 32768^2 at 8 GPUs: 4095 or 4096 output rows + 4 halo rows each (over-read 4/band)
    bands = shard.row_bands(32764, 8)
    assert {b.out_rows for b in bands} <= {4095, 4096}
    assert all(b.in_row0 + b.in_rows <= 32768 for b in bands)


def test_image_shards():
    for B in (0, 1, 5, 1024):
        for G in (1, 2, 4, 8):
            s = shard.image_shards(B, G)
            assert sum(x.images for x in s) == B
            assert [x.image0 for x in s] == sorted(x.image0 for x in s)
    assert [x.images for x in shard.image_shards(1024, 8)] == [128] * 8


def test_band_view_is_a_view():
    x = torch.arange(3 * 20 * 9, dtype=torch.float32).reshape(3, 20, 9)
    b = shard.row_bands(16, 3)[1]
    v = shard.band_view(x, b)
    assert v.data_ptr() == x[:, b.out_row0].data_ptr()
    assert v.shape == (3, b.out_rows + 4, 9)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_compute(x: torch.Tensor) -> torch.Tensor:
    from oracle import cref
    return torch.from_numpy(cref.harris_f32(np.ascontiguousarray(x.numpy())))


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import cref, synth
        # config-4 analogue: one image, row bands + 4-row halo, gathered to root
        H, W = 61, 77
        n = H - 4
        full = torch.from_numpy(synth.synth_numpy(3, H, W, seed=4242))
        bands = shard.row_bands(n, world)
        mine = bands[rank]
        local = shard.harris_row_band(shard.band_view(full, mine), compute=_oracle_compute)
        assert local.shape == (mine.out_rows, W - 4)
        got = shard.gather_rows(local, bands, root=0)
        # config-5 analogue: image shards, one batched call per rank
        B, h, w = 5, 20, 24
        imgs = synth.synth_numpy(3 * B, h, w, seed=7).reshape(B, 3, h, w)
        shards = shard.image_shards(B, world)
        s = shards[rank]
        part = torch.from_numpy(cref.harris_f32_batched(np.ascontiguousarray(imgs[s.image0:s.image0 + s.images])))
        got_b = shard.gather_images(part, shards, root=0)
        if rank == 0:
            ok_rows = np.array_equal(got.numpy(), cref.harris_f32(full.numpy()))
            ok_imgs = np.array_equal(got_b.numpy(), cref.harris_f32_batched(imgs))
            result_q.put((ok_rows, ok_imgs))
        else:
            assert got is None and got_b is None
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_shard_and_gather(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    ok_rows, ok_imgs = q.get(timeout=5)
    assert ok_rows and ok_imgs


def test_peer_gather_offsets_tile_the_result():
    """The fused gather's per-rank output offsets (peer.py) place every band / image
    shard exactly once inside the root's result."""
    from paper_2212_12035_b200 import peer
    n, m = 1076, 1916
    for G in (1, 2, 3, 8):
        covered = np.zeros(n, dtype=np.int32)
        for b in shard.row_bands(n, G):
            off = peer.band_offset_elems(b.out_row0, m)
            assert off % m == 0
            covered[off // m: off // m + b.out_rows] += 1
        assert (covered == 1).all()
        B = 1024
        seen = np.zeros(B, dtype=np.int32)
        for s in shard.image_shards(B, G):
            off = peer.image_offset_elems(s.image0, n, m)
            assert off == s.image0 * n * m
            seen[s.image0: s.image0 + s.images] += 1
        assert (seen == 1).all()
