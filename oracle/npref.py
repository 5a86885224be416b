"""Pure numpy restatement of the Harris pipeline — TEST INFRASTRUCTURE ONLY.

Direct transcription of the Halide algorithm the thesis takes as ground truth
 in the op order of SURVEY.md Appendix B, vectorised over
whole planes.  ``harris_np(rgb, dtype=np.float32)`` follows the f32 contract
(each product / sum rounded to f32, numpy never fuses); ``dtype=np.float64``
follows the sges evaluation order.  Used to cross-check the C oracle and to
evaluate known-answer images.
"""
from __future__ import annotations

import numpy as np


def harris_np(rgb: np.ndarray, kappa: float = 0.04, dtype=np.float32, window: str = "box") -> np.ndarray:
    rgb = np.asarray(rgb, dtype=np.float32)
    if rgb.ndim != 3 or rgb.shape[0] != 3 or rgb.shape[1] < 5 or rgb.shape[2] < 5:
        raise ValueError("rgb must be (3, H>=5, W>=5)")
    f = np.dtype(dtype).type
    R, G, B = (rgb[c].astype(dtype) for c in range(3))
    if dtype == np.float32:
        wg = (f(0.299), f(0.587), f(0.114))
        a, b = f(0.083333336), f(0.16666667)
    else:
        wg = (0.299, 0.587, 0.114)
        a, b = 1.0 / 12.0, 2.0 / 12.0
    z = f(0.0)
    g = ((z + wg[0] * R) + wg[1] * G) + wg[2] * B
    H, W = g.shape
    sx = ((-a, z, a), (-b, z, b), (-a, z, a))
    sy = ((-a, -b, -a), (z, z, z), (a, b, a))
    Ix = np.zeros((H - 2, W - 2), dtype=dtype)
    Iy = np.zeros((H - 2, W - 2), dtype=dtype)
    for i in range(3):
        for j in range(3):
            win = g[i:i + H - 2, j:j + W - 2]
            Ix = Ix + sx[i][j] * win
            Iy = Iy + sy[i][j] * win
    Ixx, Ixy, Iyy = Ix * Ix, Ix * Iy, Iy * Iy
    n, m = H - 4, W - 4
    Sxx = np.zeros((n, m), dtype=dtype)
    Sxy = np.zeros((n, m), dtype=dtype)
    Syy = np.zeros((n, m), dtype=dtype)
    w2d = ((1, 2, 1), (2, 4, 2), (1, 2, 1))  # binomial window (evalref.py:114-115)
    for i in range(3):
        for j in range(3):
            if window == "binomial":  # row-major w*p accumulation from 0 (f32: w*p is exact)
                w = f(w2d[i][j])
                Sxx = Sxx + w * Ixx[i:i + n, j:j + m]
                Sxy = Sxy + w * Ixy[i:i + n, j:j + m]
                Syy = Syy + w * Iyy[i:i + n, j:j + m]
            else:
                Sxx = Sxx + Ixx[i:i + n, j:j + m]
                Sxy = Sxy + Ixy[i:i + n, j:j + m]
                Syy = Syy + Iyy[i:i + n, j:j + m]
    k = f(kappa)
    det = Sxx * Syy - Sxy * Sxy
    tr = Sxx + Syy
    return (det - (k * tr) * tr).astype(dtype)


def harris_rrot_np(rgb: np.ndarray, kappa: float = 0.04) -> np.ndarray:
    """f32 restatement of the thesis's cbuf+rrot schedule's ARITHMETIC:
    separated Sobel — vertical [1,2,1] sum / [-1,0,1] difference of gray columns
    (PAPER.md:4777-4790), then the horizontal -1/12, 0, 1/12 and 1/12, 1/6, 1/12 taps
     — and box sums as vertical 3-row sums of the products followed by
    horizontal 3-sums, every accumulation from 0 in listing order.
    Independent of oracle/harris_oracle.c's line buffers; pins oracle_harris_f32_rrot."""
    rgb = np.asarray(rgb, dtype=np.float32)
    if rgb.ndim != 3 or rgb.shape[0] != 3 or rgb.shape[1] < 5 or rgb.shape[2] < 5:
        raise ValueError("rgb must be (3, H>=5, W>=5)")
    f = np.float32
    z = f(0.0)
    g = ((z + f(0.299) * rgb[0]) + f(0.587) * rgb[1]) + f(0.114) * rgb[2]
    H, W = g.shape
    g0, g1, g2 = g[0:H - 2], g[1:H - 1], g[2:H]
    vs = ((z + f(1.0) * g0) + f(2.0) * g1) + f(1.0) * g2
    vd = ((z + f(-1.0) * g0) + f(0.0) * g1) + f(1.0) * g2
    a, b = f(0.083333336), f(0.16666667)
    c0, c1, c2 = slice(0, W - 2), slice(1, W - 1), slice(2, W)
    Ix = ((z + (-a) * vs[:, c0]) + z * vs[:, c1]) + a * vs[:, c2]
    Iy = ((z + a * vd[:, c0]) + b * vd[:, c1]) + a * vd[:, c2]
    n, m = H - 4, W - 4
    r0, r1, r2 = slice(0, n), slice(1, n + 1), slice(2, n + 2)

    def vsum(p, q):
        return ((z + p[r0] * q[r0]) + p[r1] * q[r1]) + p[r2] * q[r2]

    vxx, vxy, vyy = vsum(Ix, Ix), vsum(Ix, Iy), vsum(Iy, Iy)

    def hsum(v):
        return ((z + v[:, 0:m]) + v[:, 1:m + 1]) + v[:, 2:m + 2]

    sxx, sxy, syy = hsum(vxx), hsum(vxy), hsum(vyy)
    k = f(kappa)
    return ((sxx * syy - sxy * sxy) - (k * (sxx + syy)) * (sxx + syy)).astype(np.float32)
