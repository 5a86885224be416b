"""Multi-GPU sharding of the Harris path (BASELINE.json north_star).

The path has no exchange step, so there is no per-pixel collective:

* one large image (config 4): output rows are split into contiguous bands
  ``[floor(g*n/G), floor((g+1)*n/G))``; GPU g holds input rows ``[r0, r1+4)`` —
  its band plus a 4-row halo re-read from its own copy — and runs the fused
  kernel on that strided view.  Columns are never split.
* a batch (config 5): images ``[floor(g*B/G), floor((g+1)*B/G))`` per GPU, one
  batched launch per GPU.
* the only cross-GPU traffic is the optional final gather of the output to a
  root rank (point-to-point send/recv; over NCCL that is NVLink / NVSwitch).

The thesis itself is single-device ("support for multiple devices is left for
future work"); its within-device analogue is the 32-row strip
split with a 4-row overlap, ``slide (32+4) 32``.

Everything here is plain index arithmetic plus torch.distributed plumbing; the
compute function is injectable so the CPU (gloo) tests can exercise the
partitioning with the oracle while the product path uses the fused kernel.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class RowBand:
    rank: int
    out_row0: int      # first output row of the band
    out_rows: int      # output rows in the band (may be 0 when G > n)

    @property
    def in_row0(self) -> int:
        return self.out_row0

    @property
    def in_rows(self) -> int:
        """input rows the band reads: its output rows plus the 4-row halo"""
        return self.out_rows + 4 if self.out_rows > 0 else 0


@dataclass(frozen=True)
class ImageShard:
    rank: int
    image0: int
    images: int


def row_bands(n: int, world: int) -> list[RowBand]:
    """Split n output rows into `world` contiguous bands, sizes differing by <= 1."""
    if n < 1 or world < 1:
        raise ValueError("n and world must be >= 1")
    return [RowBand(g, (g * n) // world, ((g + 1) * n) // world - (g * n) // world) for g in range(world)]


def image_shards(batch: int, world: int) -> list[ImageShard]:
    if batch < 0 or world < 1:
        raise ValueError("batch must be >= 0 and world >= 1")
    return [ImageShard(g, (g * batch) // world, ((g + 1) * batch) // world - (g * batch) // world)
            for g in range(world)]


def band_view(rgb: torch.Tensor, band: RowBand) -> torch.Tensor:
    """Input view (3, out_rows+4, W) of a (3, H, W) image for one band — no copy."""
    return rgb[:, band.in_row0: band.in_row0 + band.in_rows, :]


def default_compute(x: torch.Tensor) -> torch.Tensor:
    from .harris import harris
    return harris(x)


def harris_row_band(rgb_band: torch.Tensor, compute: Optional[Callable] = None) -> torch.Tensor:
    """Run the fused kernel on this rank's band (3, out_rows+4, W) -> (out_rows, W-4)."""
    return (compute or default_compute)(rgb_band)


def gather_rows(local: torch.Tensor, bands: list[RowBand], root: int = 0,
                group: Optional[dist.ProcessGroup] = None) -> Optional[torch.Tensor]:
    """Gather every rank's output band to `root` with point-to-point transfers
    (NVLink under NCCL); returns the full (n, m) output on root, None elsewhere."""
    rank = dist.get_rank(group)
    m = local.shape[-1]
    n = sum(b.out_rows for b in bands)
    if rank != root:
        if local.numel():
            dist.send(local.contiguous(), dst=root, group=group)
        return None
    full = torch.empty((n, m), dtype=local.dtype, device=local.device)
    reqs = []
    for b in bands:
        if b.out_rows == 0:
            continue
        dst = full[b.out_row0: b.out_row0 + b.out_rows]
        if b.rank == root:
            dst.copy_(local)
        else:
            reqs.append(dist.irecv(dst, src=b.rank, group=group))
    for r in reqs:
        r.wait()
    return full


def gather_images(local: torch.Tensor, shards: list[ImageShard], root: int = 0,
                  group: Optional[dist.ProcessGroup] = None) -> Optional[torch.Tensor]:
    """Gather (images, n, m) shards to `root`; returns (B, n, m) on root."""
    rank = dist.get_rank(group)
    if rank != root:
        if local.numel():
            dist.send(local.contiguous(), dst=root, group=group)
        return None
    B = sum(s.images for s in shards)
    full = torch.empty((B,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    reqs = []
    for s in shards:
        if s.images == 0:
            continue
        dst = full[s.image0: s.image0 + s.images]
        if s.rank == root:
            dst.copy_(local)
        else:
            reqs.append(dist.irecv(dst, src=s.rank, group=group))
    for r in reqs:
        r.wait()
    return full
