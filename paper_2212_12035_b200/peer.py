"""Fused compute + gather over peer memory (BASELINE.json north_star:
"results are gathered over NVLink only for the final output").

The gather is not a collective that runs after the kernel.  The root rank owns the
result buffer(s) and a small flag array; every rank maps them (CUDA IPC — NVLink 5 /
NVSwitch peer mappings on a multi-GPU node) and runs the fused Harris kernel with its
output pointer aimed at its own rows / images inside the root's buffer
(``harris_run_notify``), so every output row crosses the link as soon as it is produced
and the transfer overlaps the rest of the stencil.  The kernel's last CTA releases the
step's epoch into the rank's flag slot; the root's stream acquires all slots
(``harris_peer_wait``, a one-warp spin kernel with a timeout) and anything queued after
it on that stream sees the complete result.

Back-pressure: the result is multi-buffered (``buffers``, default 2).  At the start of
step e the root publishes "every stream-ordered use of step e-1 is finished" into a
release slot; a rank writing step e first waits (device side, on its own stream) until
the root released step e - buffers, so no rank can overwrite a buffer the root's
consumers are still reading.  Neither the data path nor the synchronisation involves the
host or NCCL; torch.distributed only exchanges the IPC handles once.

Flag array layout (uint32, root memory): ``[0, world)`` done-epoch per rank,
``world`` the root's released epoch.

The thesis itself is single-device; this is the B200 build's multi-GPU
extension of the thesis's output-strip partitioning.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import torch
import torch.distributed as dist

from ._lib import PeerHandle, check, lib
from .harris import KAPPA, _flags, context

DEFAULT_TIMEOUT_S = 20.0


def band_offset_elems(out_row0: int, out_pitch: int) -> int:
    """Element offset of output row ``out_row0`` in a single (n, out_pitch) result."""
    return out_row0 * out_pitch


def image_offset_elems(image0: int, n: int, m: int) -> int:
    """Element offset of image ``image0`` in a contiguous (B, n, m) result."""
    return image0 * n * m


def _export(t: torch.Tensor) -> bytes:
    h = PeerHandle()
    check(lib().harris_peer_export(t.data_ptr(), ctypes.byref(h)), "harris_peer_export")
    return h.to_bytes()


class PeerGather:
    """Result buffers on ``root``; every rank's fused kernel writes its share into them.

    ``shape``: the full result shape on root, ``(n, m)`` for a row-banded image or
    ``(B, n, m)`` for an image-sharded batch.  Collective constructor (all ranks)."""

    def __init__(self, shape: Sequence[int], root: int = 0, group: Optional[dist.ProcessGroup] = None,
                 device: Optional[int] = None, buffers: int = 2, timeout_s: float = DEFAULT_TIMEOUT_S):
        if buffers < 1:
            raise ValueError("buffers must be >= 1")
        self.shape = tuple(int(s) for s in shape)
        self.root, self.group = root, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.buffers = buffers
        self.timeout_ns = int(timeout_s * 1e9)
        self.epoch = 0
        self._mappings: list[int] = []
        dev = torch.device("cuda", self.device)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)  # wait-timeout bit (local)
        handles = None
        if self.rank == root:
            self.results = [torch.empty(self.shape, dtype=torch.float32, device=dev) for _ in range(buffers)]
            self.flags = torch.zeros(self.world + 1, dtype=torch.int32, device=dev)
            torch.cuda.synchronize(dev)
            handles = [[_export(r) for r in self.results], _export(self.flags)]
        obj = [handles]
        dist.broadcast_object_list(obj, src=root, group=group)
        res_h, flag_h = obj[0]
        if self.rank == root:
            self._res_ptrs = [r.data_ptr() for r in self.results]
            self._flags_ptr = self.flags.data_ptr()
        else:
            self.results = None
            self._res_ptrs = [self._open(h) for h in res_h]
            self._flags_ptr = self._open(flag_h)

    def _open(self, hb: bytes) -> int:
        h = PeerHandle.from_bytes(hb)
        mapping, ptr = ctypes.c_void_p(), ctypes.c_void_p()
        check(lib().harris_peer_open(self.device, ctypes.byref(h), ctypes.byref(mapping), ctypes.byref(ptr)),
              "harris_peer_open")
        self._mappings.append(mapping.value)
        return ptr.value

    # ---------------------------------------------------------------- one step
    def _begin(self, stream) -> tuple[int, int]:
        self.epoch = (self.epoch + 1) & 0xFFFFFFFF
        e = self.epoch
        L = lib()
        release_slot = self._flags_ptr + 4 * self.world
        if self.rank == self.root:
            # everything queued on this stream so far (the consumers of step e-1) is done
            check(L.harris_peer_signal(release_slot, (e - 1) & 0xFFFFFFFF, stream), "harris_peer_signal")
        else:
            # do not overwrite a buffer whose previous step the root has not released
            check(L.harris_peer_wait(release_slot, 1, (e - self.buffers) & 0xFFFFFFFF, self.status.data_ptr(),
                                     self.timeout_ns, stream), "harris_peer_wait")
        return e, self._res_ptrs[e % self.buffers]

    def _finish(self, e: int, stream) -> Optional[torch.Tensor]:
        if self.rank != self.root:
            return None
        check(lib().harris_peer_wait(self._flags_ptr, self.world, e, self.status.data_ptr(), self.timeout_ns,
                                     stream), "harris_peer_wait")
        return self.results[e % self.buffers]

    def _run(self, rgb: torch.Tensor, out_offset: int, n_local: int, m: int, out_pitch: int, out_image_stride: int,
             batch: int, kappa: float, exact: bool) -> Optional[torch.Tensor]:
        stream = torch.cuda.current_stream(self.device).cuda_stream
        e, base = self._begin(stream)
        flag = self._flags_ptr + 4 * self.rank
        if n_local == 0 or batch == 0:
            check(lib().harris_peer_signal(flag, e, stream), "harris_peer_signal")
        else:
            if rgb.dtype != torch.float32 or rgb.stride(-1) != 1 or rgb.device.index != self.device:
                raise ValueError("rgb must be float32 on this rank's device with unit column stride")
            s = rgb.stride()
            if rgb.dim() == 3:
                in_chan, in_pitch = s[0], s[1]
                in_image = 3 * in_chan
            else:
                in_image, in_chan, in_pitch = s[0], s[1], s[2]
            ctx = context(self.device)
            rc = lib().harris_run_notify(ctx.handle, base + 4 * out_offset, out_pitch, out_image_stride, n_local, m,
                                         rgb.data_ptr(), in_pitch, in_chan, in_image, batch, kappa,
                                         _flags(exact, False, False), flag, e, stream)
            check(rc, "harris_run_notify", ctx.handle)
        return self._finish(e, stream)

    def run_rows(self, rgb_band: torch.Tensor, out_row0: int, kappa: float = KAPPA,
                 exact: bool = False) -> Optional[torch.Tensor]:
        """This rank's row band ``(3, rows+4, W)`` (a view with the parent's strides is
        fine) -> rows ``[out_row0, out_row0+rows)`` of the root's ``(n, m)`` result.
        Returns the result tensor on root (valid in stream order), None elsewhere."""
        if len(self.shape) != 2:
            raise ValueError("run_rows needs a (n, m) result")
        n, m = self.shape
        rows = max(0, rgb_band.shape[-2] - 4) if rgb_band.numel() else 0
        if rows and (rgb_band.shape[-1] != m + 4 or out_row0 < 0 or out_row0 + rows > n):
            raise ValueError("band does not fit the result")
        return self._run(rgb_band, band_offset_elems(out_row0, m), rows, m, m, rows * m, 1, kappa, exact)

    def run_images(self, rgb: torch.Tensor, image0: int, kappa: float = KAPPA,
                   exact: bool = False) -> Optional[torch.Tensor]:
        """This rank's images ``(nb, 3, H, W)`` -> images ``[image0, image0+nb)`` of the
        root's ``(B, n, m)`` result."""
        if len(self.shape) != 3:
            raise ValueError("run_images needs a (B, n, m) result")
        B, n, m = self.shape
        nb = rgb.shape[0] if rgb.numel() else 0
        if nb and (tuple(rgb.shape[1:]) != (3, n + 4, m + 4) or image0 < 0 or image0 + nb > B):
            raise ValueError("images do not fit the result")
        return self._run(rgb, image_offset_elems(image0, n, m), n if nb else 0, m, m, n * m, nb, kappa, exact)

    def check(self) -> None:
        """Synchronise this rank's device and raise if a wait timed out."""
        torch.cuda.synchronize(self.device)
        if int(self.status.item()) != 0:
            raise RuntimeError("peer gather: a flag wait timed out (a peer did not finish its step)")

    def close(self) -> None:
        """Collective: unmap the root's buffers on every rank before the root frees them."""
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        for mp in self._mappings:
            lib().harris_peer_close(self.device, mp)
        self._mappings = []
        dist.barrier(group=self.group)
