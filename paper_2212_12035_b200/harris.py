"""PyTorch-facing mirror of the thesis Harris boundary, backed by the C-ABI.

``harris(rgb)`` is the Rise ``harris : 3.(n+4).(m+4).f32 -> n.m.f32``
(PAPER.md:2482-2496): planar RGB in, the valid region (4 smaller in each
dimension, no padding) out.  A leading batch dimension is accepted.  CUDA
tensors run on the current stream with no host synchronisation; CPU tensors /
numpy arrays go through ``harris_run_host`` (pipelined H2D -> fused kernel ->
D2H on the device), never through a CPU implementation.

Torch is plumbing here (device memory, streams); the arithmetic is in
``csrc/harris_tma.cu`` / ``csrc/harris_generic.cu``.
"""
from __future__ import annotations

import ctypes
import threading
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import FLAG_EXACT_ORDER, FLAG_FORCE_GENERIC, FLAG_FORCE_TMA, PlanInfo, check, lib

KAPPA = 0.04


class HarrisContext:
    """One ``harris_ctx`` bound to a CUDA device (``harris_init_ex`` / ``harris_destroy``).

    ``l2_policy`` (``_lib.L2_EVICT_*``), ``band_rows`` and ``pdl`` map to ``harris_options``; None
    keeps the library default (evict_last input loads, planner-chosen tiles, PDL launches)."""

    def __init__(self, device: int, l2_policy: Optional[int] = None, band_rows: Optional[int] = None,
                 pdl: Optional[bool] = None):
        self.device = int(device)
        h = ctypes.c_void_p()
        opts = _lib.Options()
        lib().harris_options_default(ctypes.byref(opts))
        if l2_policy is not None:
            opts.l2_policy = int(l2_policy)
        if band_rows is not None:
            opts.band_rows = int(band_rows)
        if pdl is not None:
            opts.pdl = 1 if pdl else 0
        check(lib().harris_init_ex(ctypes.byref(h), self.device, ctypes.byref(opts)),
              f"harris_init_ex(cuda:{self.device})")
        self._h = h

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().harris_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    @property
    def last_path(self) -> int:
        return int(lib().harris_last_path(self._h))

    @property
    def num_sms(self) -> int:
        return int(lib().harris_num_sms(self._h))

    def run_strided(self, out_ptr: int, out_pitch: int, out_image_stride: int, n: int, m: int, rgb_ptr: int,
                    in_pitch: int, in_chan_stride: int, in_image_stride: int, batch: int,
                    kappa: float = KAPPA, flags: int = 0, stream: int = 0) -> None:
        rc = lib().harris_run_strided(self._h, out_ptr, out_pitch, out_image_stride, n, m, rgb_ptr, in_pitch,
                                      in_chan_stride, in_image_stride, batch, kappa, flags, stream)
        check(rc, "harris_run_strided", self._h)

    def plan(self, n: int, m: int, batch: int = 1, rgb_ptr: int = 0, in_pitch: Optional[int] = None,
             in_chan_stride: Optional[int] = None, in_image_stride: Optional[int] = None, out_ptr: int = 0,
             out_pitch: Optional[int] = None, out_image_stride: Optional[int] = None, flags: int = 0) -> dict:
        W, H = m + 4, n + 4
        in_pitch = W if in_pitch is None else in_pitch
        in_chan_stride = H * in_pitch if in_chan_stride is None else in_chan_stride
        in_image_stride = 3 * in_chan_stride if in_image_stride is None else in_image_stride
        out_pitch = m if out_pitch is None else out_pitch
        out_image_stride = n * out_pitch if out_image_stride is None else out_image_stride
        # a dummy 256-byte aligned address stands in for "some aligned buffer"
        rgb_ptr = rgb_ptr or 1 << 20
        out_ptr = out_ptr or 1 << 21
        info = PlanInfo()
        rc = lib().harris_plan(self._h, n, m, batch, rgb_ptr, in_pitch, in_chan_stride, in_image_stride,
                               out_ptr, out_pitch, out_image_stride, flags, ctypes.byref(info))
        check(rc, "harris_plan", self._h)
        return info.as_dict()

    def run_host(self, rgb: np.ndarray, out: Optional[np.ndarray] = None, kappa: float = KAPPA,
                 flags: int = 0) -> np.ndarray:
        """Host buffers in, host buffer out (pinned memory gives full PCIe speed)."""
        if rgb.dtype != np.float32 or not rgb.flags.c_contiguous:
            raise ValueError("rgb must be C-contiguous float32")
        batched = rgb.ndim == 4
        x = rgb if batched else rgb[None]
        if x.ndim != 4 or x.shape[1] != 3:
            raise ValueError("rgb must be (3, H, W) or (B, 3, H, W)")
        B, _, H, W = x.shape
        n, m = H - 4, W - 4
        if out is None:
            out = np.empty((B, n, m) if batched else (n, m), dtype=np.float32)
        if out.dtype != np.float32 or not out.flags.c_contiguous or out.size != B * max(n, 0) * max(m, 0):
            raise ValueError("out must be C-contiguous float32 of the output shape")
        rc = lib().harris_run_host(self._h, out.ctypes.data, m, n, m, x.ctypes.data, B, kappa, flags)
        check(rc, "harris_run_host", self._h)
        return out


_ctx_lock = threading.Lock()
_contexts: dict[int, HarrisContext] = {}


def context(device: Optional[int] = None) -> HarrisContext:
    """The process-wide context of a CUDA device (created on first use)."""
    dev = torch.cuda.current_device() if device is None else int(device)
    c = _contexts.get(dev)
    if c is not None:
        return c
    with _ctx_lock:
        c = _contexts.get(dev)
        if c is None:
            c = HarrisContext(dev)
            _contexts[dev] = c
        return c


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_handle(dev: int, stream: Optional[torch.cuda.Stream]) -> int:
    """cudaStream_t of `stream` or of the device's current stream (the raw query avoids
    building a Stream object per call: this is on the per-launch host path)."""
    if stream is not None:
        return stream.cuda_stream
    if _raw_stream is not None:
        return _raw_stream(dev)
    return torch.cuda.current_stream(dev).cuda_stream


WINDOWS = ("box", "binomial")


def _window_flag(window: str) -> int:
    """window "box": the thesis's 3x3 '+' sums; "binomial": the reference's weights2d window
    (HARRIS_FLAG_BINOMIAL_WINDOW)."""
    if window not in WINDOWS:
        raise ValueError(f"window must be one of {WINDOWS}")
    return _lib.FLAG_BINOMIAL_WINDOW if window == "binomial" else 0


def _flags(exact: bool, force_generic: bool, force_tma: bool, pdl=False) -> int:
    """pdl: False; True = HARRIS_FLAG_PDL (prologue overlaps the previous kernel, waits before
    touching memory); "independent" = HARRIS_FLAG_PDL_INDEPENDENT (the caller guarantees the
    still-running stream work neither writes this call's input nor touches its output)."""
    if pdl not in (False, True, "independent"):
        raise ValueError('pdl must be False, True or "independent"')
    return (FLAG_EXACT_ORDER if exact else 0) | (FLAG_FORCE_GENERIC if force_generic else 0) | (
        FLAG_FORCE_TMA if force_tma else 0) | (_lib.FLAG_PDL if pdl is True else 0) | (
        _lib.FLAG_PDL_INDEPENDENT if pdl == "independent" else 0)


def _check_rgb(rgb) -> tuple[int, int, int]:
    if rgb.dtype not in (torch.float32, np.float32):
        raise TypeError("harris expects float32 planar RGB (Rise type 3.(n+4).(m+4).f32)")
    shape = tuple(rgb.shape)
    if len(shape) == 3:
        B = 1
        C, H, W = shape
    elif len(shape) == 4:
        B, C, H, W = shape
    else:
        raise ValueError("rgb must be (3, H, W) or (B, 3, H, W)")
    if C != 3:
        raise ValueError(f"expected 3 planar channels, got {C}")
    if H < 5 or W < 5:
        raise ValueError(f"harris needs an input of at least 5x5, got {H}x{W}")
    return B, H, W


def harris(rgb, kappa: float = KAPPA, *, out: Optional[torch.Tensor] = None, exact: bool = False,
           force_generic: bool = False, force_tma: bool = False, stream: Optional[torch.cuda.Stream] = None,
           ctx: Optional[HarrisContext] = None, pdl=False, window: str = "box"):
    """Fused Harris coarsity of planar RGB f32.

    rgb: ``(3, H, W)`` or ``(B, 3, H, W)`` float32; CUDA tensor (device path,
    asynchronous on ``stream`` / the current stream) or CPU tensor / numpy array
    (host path through the device).  Returns ``(H-4, W-4)`` / ``(B, H-4, W-4)``.
    ``exact=True`` selects the Appendix-B op order (bit-identical to the C
    oracle); the default is the FMA/separable order, within the SURVEY.md §8(d)
    tolerance of the f64 reference.  ``pdl`` (device path): programmatic dependent launch for
    back-to-back frame streams (see ``_flags``).  ``window="binomial"``: the binomial
    window in place of the 3x3 box sums (``_window_flag``).
    """
    flags = _flags(exact, force_generic, force_tma, pdl) | _window_flag(window)
    if isinstance(rgb, np.ndarray) or (isinstance(rgb, torch.Tensor) and not rgb.is_cuda):
        _check_rgb(rgb)
        arr = rgb if isinstance(rgb, np.ndarray) else rgb.numpy()
        arr = np.ascontiguousarray(arr)
        dev = torch.cuda.current_device()
        host_out = None
        if out is not None:  # a host array / CPU tensor of the output shape (pinned for full speed)
            host_out = out if isinstance(out, np.ndarray) else out.numpy()
        res = context(dev).run_host(arr, out=host_out, kappa=kappa, flags=flags)
        if out is not None:
            return out
        return res if isinstance(rgb, np.ndarray) else torch.from_numpy(res)
    B, H, W = _check_rgb(rgb)
    if rgb.stride(-1) != 1:
        rgb = rgb.contiguous()
    n, m = H - 4, W - 4
    batched = rgb.dim() == 4
    if out is None:
        out = torch.empty((B, n, m) if batched else (n, m), dtype=torch.float32, device=rgb.device)
    else:
        if out.dtype != torch.float32 or out.device != rgb.device:
            raise ValueError("out must be float32 on the input's device")
        if tuple(out.shape) != ((B, n, m) if batched else (n, m)) or out.stride(-1) != 1:
            raise ValueError("out has the wrong shape or a non-unit column stride")
    s_in = rgb.stride()
    s_out = out.stride()
    if batched:
        in_image, in_chan, in_pitch = s_in[0], s_in[1], s_in[2]
        out_image, out_pitch = s_out[0], s_out[1]
    else:
        in_chan, in_pitch = s_in[0], s_in[1]
        in_image = 3 * in_chan
        out_pitch = s_out[0]
        out_image = n * out_pitch
    dev = rgb.device.index if rgb.device.index is not None else torch.cuda.current_device()
    (ctx or context(dev)).run_strided(out.data_ptr(), out_pitch, out_image, n, m, rgb.data_ptr(), in_pitch,
                                      in_chan, in_image, B, kappa, flags, _stream_handle(dev, stream))
    return out


def harris_frames(frames, outs=None, kappa: float = KAPPA, *, exact: bool = False, independent: bool = False,
                  stream: Optional[torch.cuda.Stream] = None, ctx: Optional[HarrisContext] = None):
    """A stream of independent single frames through ``harris_run_frames`` (planar f32) or
    ``harris_run_frames_u8`` (interleaved uint8): one launch per frame, back to back, chained
    with programmatic dependent launch (frame 0 waits for earlier stream work unless
    ``independent``).  ``frames``: (3, H, W) float32 or (H, W, 3) uint8 CUDA tensors of one shape
    and layout (same strides); ``outs``: matching (H-4, W-4) outputs (allocated when None), all
    distinct.  Returns ``outs``."""
    frames = list(frames)
    if not frames:
        raise ValueError("no frames")
    f0 = frames[0]
    u8 = f0.dtype == torch.uint8
    if u8:
        if f0.dim() != 3 or f0.shape[-1] != 3 or not f0.is_cuda or f0.stride(-1) != 1 or f0.stride(-2) != 3:
            raise ValueError("u8 frames must be (H, W, 3) interleaved CUDA tensors")
        H, W = f0.shape[0], f0.shape[1]
        if H < 5 or W < 5:
            raise ValueError(f"harris needs an input of at least 5x5, got {H}x{W}")
    else:
        _check_rgb(f0)
        if f0.dim() != 3 or not f0.is_cuda or f0.stride(-1) != 1:
            raise ValueError("frames must be (3, H, W) CUDA tensors with unit column stride")
        H, W = f0.shape[1], f0.shape[2]
    for f in frames:
        if f.shape != f0.shape or f.stride() != f0.stride() or f.dtype != f0.dtype or f.device != f0.device:
            raise ValueError("all frames must share shape, strides, dtype and device")
    n, m = H - 4, W - 4
    if outs is None:
        outs = [torch.empty((n, m), dtype=torch.float32, device=f0.device) for _ in frames]
    outs = list(outs)
    if len(outs) != len(frames):
        raise ValueError("one output per frame")
    o0 = outs[0]
    for o in outs:
        if o.shape != (n, m) or o.dtype != torch.float32 or o.device != f0.device or o.stride() != o0.stride() or \
                o.stride(-1) != 1:
            raise ValueError("outputs must be float32 (H-4, W-4) tensors on the frames' device with one row pitch")
    if len({o.data_ptr() for o in outs}) != len(outs):
        raise ValueError("outputs must be distinct")
    dev = f0.device.index if f0.device.index is not None else torch.cuda.current_device()
    vp = ctypes.c_void_p
    optrs = (vp * len(outs))(*[o.data_ptr() for o in outs])
    iptrs = (vp * len(frames))(*[f.data_ptr() for f in frames])
    flags = _flags(exact, False, False, "independent" if independent else False)
    ctx = ctx or context(dev)
    if u8:
        rc = lib().harris_run_frames_u8(ctx.handle, optrs, o0.stride(0), n, m, iptrs, f0.stride(0), len(frames),
                                        kappa, flags, _stream_handle(dev, stream))
        check(rc, "harris_run_frames_u8", ctx.handle)
    else:
        rc = lib().harris_run_frames(ctx.handle, optrs, o0.stride(0), n, m, iptrs, f0.stride(1), f0.stride(0),
                                     len(frames), kappa, flags, _stream_handle(dev, stream))
        check(rc, "harris_run_frames", ctx.handle)
    return outs


def harris_u8(rgb8, kappa: float = KAPPA, *, out: Optional[torch.Tensor] = None, exact: bool = False,
              force_generic: bool = False, force_tma: bool = False, stream: Optional[torch.cuda.Stream] = None,
              ctx: Optional[HarrisContext] = None, pdl=False, window: str = "box"):
    """Fused Harris on interleaved 8-bit RGB: ``(H, W, 3)`` or ``(B, H, W, 3)`` uint8
    (value/255), CUDA (device path) or CPU/numpy (host path through the device).
    Returns ``(H-4, W-4)`` / ``(B, H-4, W-4)`` float32, equal to ``harris`` on the planar
    image ``rgb8/255`` (bit-for-bit with ``exact=True``)."""
    flags = _flags(exact, force_generic, force_tma, pdl) | _window_flag(window)
    shape = tuple(rgb8.shape)
    if rgb8.dtype not in (torch.uint8, np.uint8):
        raise TypeError("harris_u8 expects uint8 interleaved RGB")
    if len(shape) not in (3, 4) or shape[-1] != 3:
        raise ValueError("rgb8 must be (H, W, 3) or (B, H, W, 3)")
    H, W = shape[-3], shape[-2]
    if H < 5 or W < 5:
        raise ValueError(f"harris needs an input of at least 5x5, got {H}x{W}")
    B = shape[0] if len(shape) == 4 else 1
    n, m = H - 4, W - 4
    batched = len(shape) == 4
    if isinstance(rgb8, np.ndarray) or not rgb8.is_cuda:
        arr = np.ascontiguousarray(rgb8 if isinstance(rgb8, np.ndarray) else rgb8.numpy())
        oshape = (B, n, m) if batched else (n, m)
        if out is not None:  # a host array / CPU tensor of the output shape (pinned for full speed)
            res = out if isinstance(out, np.ndarray) else out.numpy()
            if res.dtype != np.float32 or res.shape != oshape or not res.flags["C_CONTIGUOUS"]:
                raise ValueError("out must be a C-contiguous float32 host array of the output shape")
        else:
            res = np.empty(oshape, dtype=np.float32)
        ctx = ctx or context(torch.cuda.current_device())
        rc = lib().harris_run_host_u8(ctx.handle, res.ctypes.data, m, n, m, arr.ctypes.data, B, kappa, flags)
        check(rc, "harris_run_host_u8", ctx.handle)
        if out is not None:
            return out
        return res if isinstance(rgb8, np.ndarray) else torch.from_numpy(res)
    if rgb8.stride(-1) != 1 or rgb8.stride(-2) != 3:
        rgb8 = rgb8.contiguous()
    if out is None:
        out = torch.empty((B, n, m) if batched else (n, m), dtype=torch.float32, device=rgb8.device)
    elif tuple(out.shape) != ((B, n, m) if batched else (n, m)) or out.stride(-1) != 1 or \
            out.dtype != torch.float32 or out.device != rgb8.device:
        raise ValueError("out has the wrong shape, dtype, device or column stride")
    in_pitch = rgb8.stride(-3)
    in_image = rgb8.stride(0) if batched else H * in_pitch
    out_pitch = out.stride(-2)
    out_image = out.stride(0) if batched else n * out_pitch
    dev = rgb8.device.index if rgb8.device.index is not None else torch.cuda.current_device()
    ctx = ctx or context(dev)
    rc = lib().harris_run_u8(ctx.handle, out.data_ptr(), out_pitch, out_image, n, m, rgb8.data_ptr(), in_pitch,
                             in_image, B, kappa, flags, _stream_handle(dev, stream))
    check(rc, "harris_run_u8", ctx.handle)
    return out


BINOMIAL = (1.0, 2.0, 1.0)  # weightsV = weightsH of the reference (evalref.py:112-115)


def stencil3x3_sep(img: torch.Tensor, wv=BINOMIAL, wh=BINOMIAL, *, out: Optional[torch.Tensor] = None,
                   exact: bool = False, force_generic: bool = False, force_tma: bool = False,
                   stream: Optional[torch.cuda.Stream] = None, ctx: Optional[HarrisContext] = None,
                   pdl=False) -> torch.Tensor:
    """Separable 3x3 stencil ``(H, W)`` / ``(B, H, W)`` float32 CUDA -> ``(H-2, W-2)`` /
    ``(B, H-2, W-2)``: vertical ``wv`` then horizontal ``wh`` (the separated form of the
    reference's binomial rewrite goal)."""
    if img.dtype != torch.float32 or not img.is_cuda or img.dim() not in (2, 3):
        raise ValueError("img must be a (H, W) or (B, H, W) float32 CUDA tensor")
    H, W = img.shape[-2:]
    if H < 3 or W < 3:
        raise ValueError("stencil3x3 needs at least 3x3")
    if img.stride(-1) != 1:
        img = img.contiguous()
    batched = img.dim() == 3
    B = img.shape[0] if batched else 1
    n, m = H - 2, W - 2
    if out is None:
        out = torch.empty((B, n, m) if batched else (n, m), dtype=torch.float32, device=img.device)
    elif tuple(out.shape) != ((B, n, m) if batched else (n, m)) or out.stride(-1) != 1 or \
            out.dtype != torch.float32 or out.device != img.device:
        raise ValueError("out must be float32 on the input's device, of shape (B,) H-2, W-2 with unit column stride")
    fwv = (ctypes.c_float * 3)(*[float(v) for v in wv])
    fwh = (ctypes.c_float * 3)(*[float(v) for v in wh])
    dev = img.device.index if img.device.index is not None else torch.cuda.current_device()
    ctx = ctx or context(dev)
    rc = lib().harris_stencil3x3_sep(ctx.handle, out.data_ptr(), out.stride(-2),
                                     out.stride(0) if batched else n * out.stride(-2), n, m, img.data_ptr(),
                                     img.stride(-2), img.stride(0) if batched else H * img.stride(-2), B,
                                     fwv, fwh, _flags(exact, force_generic, force_tma, pdl),
                                     _stream_handle(dev, stream))
    check(rc, "harris_stencil3x3_sep", ctx.handle)
    return out


GROUPINGS = {
    1: "[Sx],[Sy],[x],[+],[coarsity]",
    2: "[Sx,Sy,x],[+,coarsity]",
    3: "[Sx,Sy],[x,+,coarsity]",
    4: "[Sx,Sy,x,+,coarsity]",
}


def grouping_hbm_bytes(grouping: int, n: int, m: int) -> int:
    """Compulsory HBM bytes of one image under a kernel grouping (each group reads its
    inputs once and writes its outputs once; stencil halos ignored)."""
    H, W, s, o = n + 4, m + 4, (n + 2) * (m + 2), n * m
    rgb = 12 * H * W
    return {
        1: (rgb + 4 * s) + (rgb + 4 * s) + (8 * s + 12 * s) + (12 * s + 12 * o) + (12 * o + 4 * o),
        2: (rgb + 12 * s) + (12 * s + 4 * o),
        3: (rgb + 8 * s) + (8 * s + 4 * o),
        4: rgb + 4 * o,
    }[grouping]


def harris_grouping(rgb: torch.Tensor, grouping: int, kappa: float = KAPPA, *, out: Optional[torch.Tensor] = None,
                    scratch: Optional[torch.Tensor] = None, exact: bool = False) -> torch.Tensor:
    """The thesis's kernel-grouping design space on one contiguous
    (3, H, W) CUDA image; groupings 1-3 round-trip intermediates through HBM scratch.
    FAST (default): every group is a strip-engine kernel in the fused kernel's arithmetic
    (grouping 3 is bit-identical to the fused FAST output, 1 and 2 round the products they
    materialise); ``exact=True``: the Appendix-B one-thread-per-pixel kernels (bit-identical to
    the oracle)."""
    B, H, W = _check_rgb(rgb)
    if rgb.dim() != 3 or not rgb.is_cuda or not rgb.is_contiguous():
        raise ValueError("harris_grouping takes one contiguous (3, H, W) CUDA image")
    n, m = H - 4, W - 4
    L = lib()
    need = int(L.harris_grouping_scratch_bytes(grouping, n, m))
    if need < 0:
        raise ValueError(f"unknown grouping {grouping}")
    if scratch is None and need > 0:
        scratch = torch.empty(need // 4, dtype=torch.float32, device=rgb.device)
    elif scratch is not None and (not scratch.is_contiguous() or scratch.device != rgb.device):
        raise ValueError("scratch must be a contiguous tensor on the input's device")
    if out is None:
        out = torch.empty((n, m), dtype=torch.float32, device=rgb.device)
    elif out.dtype != torch.float32 or out.device != rgb.device or tuple(out.shape) != (n, m) or \
            not out.is_contiguous():
        raise ValueError("out must be a contiguous float32 (H-4, W-4) tensor on the input's device")
    dev = rgb.device.index
    ctx = context(dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    rc = L.harris_run_grouping(ctx.handle, grouping, out.data_ptr(), n, m, rgb.data_ptr(),
                               scratch.data_ptr() if scratch is not None else None,
                               scratch.numel() * scratch.element_size() if scratch is not None else 0, kappa,
                               FLAG_EXACT_ORDER if exact else 0, st)
    check(rc, "harris_run_grouping", ctx.handle)
    return out


def synth_(dst: torch.Tensor, seed: int, dist: int = 0, *, H_global: Optional[int] = None, row0: int = 0,
           plane0: int = 0, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Fill ``dst`` (planes, rows, W) float32 CUDA, unit column stride, with the
    synthetic image stack (see ``harris_synth_fill``); returns ``dst``."""
    if dst.dtype != torch.float32 or not dst.is_cuda or dst.dim() != 3 or dst.stride(-1) != 1:
        raise ValueError("dst must be a (planes, rows, W) float32 CUDA tensor with unit column stride")
    P, R, W = dst.shape
    Hg = R if H_global is None else H_global
    st = stream if stream is not None else torch.cuda.current_stream(dst.device)
    with torch.cuda.device(dst.device):
        rc = lib().harris_synth_fill(dst.data_ptr(), P, R, W, dst.stride(1), dst.stride(0), Hg, row0, plane0,
                                     seed, dist, st.cuda_stream)
    check(rc, "harris_synth_fill")
    return dst


def algorithmic_bytes(n: int, m: int, batch: int = 1) -> int:
    """12 B read per input pixel + 4 B written per output pixel (BASELINE.json)."""
    return batch * (12 * (n + 4) * (m + 4) + 4 * n * m)


__all__ = ["HarrisContext", "context", "harris", "harris_frames", "harris_u8", "stencil3x3_sep", "BINOMIAL", "harris_grouping", "grouping_hbm_bytes", "GROUPINGS", "synth_",
           "algorithmic_bytes", "KAPPA", "_lib"]
