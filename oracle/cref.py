"""ctypes binding of ``oracle/liboracle_harris.so`` — TEST INFRASTRUCTURE ONLY.

The library is the C restatement in ``harris_oracle.c`` (f32 Appendix-B order,
f64 sges order).  ``build()`` in ``__graft_entry__`` compiles it with
``make -C oracle``; the built ``.so`` travels to the GPU box with the snapshot.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle_harris.so")

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or (
            os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "harris_oracle.c"))):
        subprocess.run(["make", "-C", _HERE, "-B" if force else "all"], check=True,
                       stdout=subprocess.DEVNULL)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        i64, fp, dp, vp = ctypes.c_int64, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double), ctypes.c_void_p
        L.oracle_harris_f32.argtypes = [vp, i64, i64, i64, vp, i64, i64, ctypes.c_float, ctypes.c_int]
        L.oracle_harris_f32.restype = ctypes.c_int
        L.oracle_harris_f64.argtypes = [vp, i64, i64, i64, vp, i64, i64, ctypes.c_double, ctypes.c_int]
        L.oracle_harris_f64.restype = ctypes.c_int
        L.oracle_harris_f32_window.argtypes = [vp, i64, i64, i64, vp, i64, i64, ctypes.c_float, ctypes.c_int,
                                                ctypes.c_int]
        L.oracle_harris_f32_window.restype = ctypes.c_int
        L.oracle_harris_f64_window.argtypes = [vp, i64, i64, i64, vp, i64, i64, ctypes.c_double, ctypes.c_int,
                                                ctypes.c_int]
        L.oracle_harris_f64_window.restype = ctypes.c_int
        L.oracle_harris_f32_batched.argtypes = [vp, i64, i64, vp, i64, ctypes.c_float, ctypes.c_int]
        L.oracle_harris_f32_batched.restype = ctypes.c_int
        L.oracle_harris_f32_rrot.argtypes = [vp, i64, i64, i64, vp, i64, i64, ctypes.c_float, ctypes.c_int]
        L.oracle_harris_f32_rrot.restype = ctypes.c_int
        L.oracle_harris_f32_rrot_batched.argtypes = [vp, i64, i64, vp, i64, ctypes.c_float, ctypes.c_int]
        L.oracle_harris_f32_rrot_batched.restype = ctypes.c_int
        L.oracle_sep3x3_f32.argtypes = [vp, i64, i64, i64, vp, i64, vp, vp, ctypes.c_int]
        L.oracle_sep3x3_f32.restype = ctypes.c_int
        L.oracle_sep3x3_f64.argtypes = [vp, i64, i64, i64, vp, i64, vp, vp, ctypes.c_int, ctypes.c_int]
        L.oracle_sep3x3_f64.restype = ctypes.c_int
        L.oracle_synth_fill.argtypes = [vp, i64, i64, i64, i64, i64, i64, i64, i64, ctypes.c_uint64, ctypes.c_int]
        L.oracle_synth_fill.restype = None
        L.oracle_max_threads.argtypes = []
        L.oracle_max_threads.restype = ctypes.c_int
        del fp, dp
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _check_rgb(rgb: np.ndarray) -> tuple[int, int]:
    if rgb.dtype != np.float32 or rgb.ndim != 3 or rgb.shape[0] != 3:
        raise ValueError("rgb must be float32 of shape (3, H, W)")
    H, W = rgb.shape[1:]
    if H < 5 or W < 5:
        raise ValueError("harris needs H >= 5 and W >= 5")
    return H, W


WINDOWS = {"box": 0, "binomial": 1}


def harris_f32(rgb: np.ndarray, kappa: float = 0.04, nthreads: int = 0, window: str = "box") -> np.ndarray:
    """f32 Appendix-B restatement. ``rgb``: (3, H, W) float32 -> (H-4, W-4) f32.
    ``window``: "box" (the thesis's 3x3 '+') or "binomial" (weights2d)."""
    rgb = np.ascontiguousarray(rgb)
    H, W = _check_rgb(rgb)
    out = np.empty((H - 4, W - 4), dtype=np.float32)
    rc = lib().oracle_harris_f32_window(_ptr(out), W - 4, H - 4, W - 4, _ptr(rgb), W, H * W, kappa, nthreads,
                                        WINDOWS[window])
    if rc:
        raise RuntimeError(f"oracle_harris_f32 failed ({rc})")
    return out


def harris_f32_rrot(rgb: np.ndarray, kappa: float = 0.04, nthreads: int = 0) -> np.ndarray:
    """Thesis cbuf+rrot schedule (separable order) in f32."""
    rgb = np.ascontiguousarray(rgb)
    H, W = _check_rgb(rgb)
    out = np.empty((H - 4, W - 4), dtype=np.float32)
    rc = lib().oracle_harris_f32_rrot(_ptr(out), W - 4, H - 4, W - 4, _ptr(rgb), W, H * W, kappa, nthreads)
    if rc:
        raise RuntimeError(f"oracle_harris_f32_rrot failed ({rc})")
    return out


def harris_f64(rgb: np.ndarray, kappa: float = 0.04, nthreads: int = 0, window: str = "box") -> np.ndarray:
    """f64 restatement in sges evaluation order, from the f32 input."""
    rgb = np.ascontiguousarray(rgb)
    H, W = _check_rgb(rgb)
    out = np.empty((H - 4, W - 4), dtype=np.float64)
    rc = lib().oracle_harris_f64_window(_ptr(out), W - 4, H - 4, W - 4, _ptr(rgb), W, H * W, kappa, nthreads,
                                        WINDOWS[window])
    if rc:
        raise RuntimeError(f"oracle_harris_f64 failed ({rc})")
    return out


def harris_f32_batched(rgb: np.ndarray, kappa: float = 0.04, nthreads: int = 0,
                       out: np.ndarray | None = None) -> np.ndarray:
    """(B, 3, H, W) float32 -> (B, H-4, W-4) float32."""
    if rgb.dtype != np.float32 or rgb.ndim != 4 or rgb.shape[1] != 3 or not rgb.flags.c_contiguous:
        raise ValueError("rgb must be C-contiguous float32 of shape (B, 3, H, W)")
    B, _, H, W = rgb.shape
    if out is None:
        out = np.empty((B, H - 4, W - 4), dtype=np.float32)
    rc = lib().oracle_harris_f32_batched(_ptr(out), H - 4, W - 4, _ptr(rgb), B, kappa, nthreads)
    if rc:
        raise RuntimeError(f"oracle_harris_f32_batched failed ({rc})")
    return out


def harris_batched(rgb: np.ndarray, variant: str = "cbuf", kappa: float = 0.04, nthreads: int = 0,
                   out: np.ndarray | None = None) -> np.ndarray:
    """Batched CPU Harris with the thesis schedule `variant` in {"cbuf", "rrot"}."""
    if variant == "cbuf":
        return harris_f32_batched(rgb, kappa, nthreads, out)
    if rgb.dtype != np.float32 or rgb.ndim != 4 or rgb.shape[1] != 3 or not rgb.flags.c_contiguous:
        raise ValueError("rgb must be C-contiguous float32 of shape (B, 3, H, W)")
    B, _, H, W = rgb.shape
    if out is None:
        out = np.empty((B, H - 4, W - 4), dtype=np.float32)
    rc = lib().oracle_harris_f32_rrot_batched(_ptr(out), H - 4, W - 4, _ptr(rgb), B, kappa, nthreads)
    if rc:
        raise RuntimeError(f"oracle_harris_f32_rrot_batched failed ({rc})")
    return out


def sep3x3_f32(img: np.ndarray, wv=(1.0, 2.0, 1.0), wh=(1.0, 2.0, 1.0), nthreads: int = 0) -> np.ndarray:
    """Separable 3x3 stencil, f32, vertical-then-horizontal order: (n+2, m+2) -> (n, m)."""
    img = np.ascontiguousarray(img, dtype=np.float32)
    if img.ndim != 2 or img.shape[0] < 3 or img.shape[1] < 3:
        raise ValueError("img must be 2-D and at least 3x3")
    n, m = img.shape[0] - 2, img.shape[1] - 2
    out = np.empty((n, m), dtype=np.float32)
    a = np.asarray(wv, dtype=np.float32)
    b = np.asarray(wh, dtype=np.float32)
    rc = lib().oracle_sep3x3_f32(_ptr(out), m, n, m, _ptr(img), m + 2, _ptr(a), _ptr(b), nthreads)
    if rc:
        raise RuntimeError(f"oracle_sep3x3_f32 failed ({rc})")
    return out


def sep3x3_f64(img: np.ndarray, wv=(1.0, 2.0, 1.0), wh=(1.0, 2.0, 1.0), form: int = 1,
               nthreads: int = 0) -> np.ndarray:
    """f64 in the reference evaluator's order: form 0 direct 2-D dot, form 1 vertical-then-horizontal."""
    img = np.ascontiguousarray(img, dtype=np.float32)
    n, m = img.shape[0] - 2, img.shape[1] - 2
    out = np.empty((n, m), dtype=np.float64)
    a = np.asarray(wv, dtype=np.float64)
    b = np.asarray(wh, dtype=np.float64)
    rc = lib().oracle_sep3x3_f64(_ptr(out), m, n, m, _ptr(img), m + 2, _ptr(a), _ptr(b), form, nthreads)
    if rc:
        raise RuntimeError(f"oracle_sep3x3_f64 failed ({rc})")
    return out


def synth(planes: int, H: int, W: int, seed: int, dist: int = 0, row0: int = 0,
          rows: int | None = None, plane0: int = 0, H_global: int | None = None) -> np.ndarray:
    rows = H if rows is None else rows
    Hg = H if H_global is None else H_global
    out = np.empty((planes, rows, W), dtype=np.float32)
    lib().oracle_synth_fill(_ptr(out), planes, rows, W, W, rows * W, Hg, row0, plane0, seed, dist)
    return out


def max_threads() -> int:
    return int(lib().oracle_max_threads())
