"""OpenCV-composed Harris — TEST INFRASTRUCTURE / REPORTED BASELINE ONLY.

The thesis compares its generated kernels against "an OpenCV-composed pipeline"
(OpenCV 4.3; Shine cbuf+rrot up to 16x faster, geomean 9.48x on
ARM).  This is the same composition with the image's OpenCV (4.13):
gray, `cv2.Sobel` (ksize 3, scale 1/12 = the Halide/thesis kernel),
products, un-normalised 3x3 `cv2.boxFilter`, coarsity; the valid region
 is cropped from OpenCV's border-replicated result.  It meets the
SURVEY.md §8(d) tolerance against the f64 oracle (tests/test_oracle.py) and is timed by
bench.py as an informational CPU point, never as the product.
"""
from __future__ import annotations

import numpy as np


def available() -> bool:
    try:
        import cv2  # noqa: F401
        return True
    except Exception:
        return False


def harris_opencv(rgb: np.ndarray, kappa: float = 0.04) -> np.ndarray:
    """(3, H, W) float32 -> (H-4, W-4) float32."""
    import cv2
    r, g, b = rgb
    gray = cv2.addWeighted(cv2.addWeighted(r, 0.299, g, 0.587, 0.0), 1.0, b, 0.114, 0.0)
    ix = cv2.Sobel(gray, cv2.CV_32F, 1, 0, ksize=3, scale=1.0 / 12.0, borderType=cv2.BORDER_REPLICATE)
    iy = cv2.Sobel(gray, cv2.CV_32F, 0, 1, ksize=3, scale=1.0 / 12.0, borderType=cv2.BORDER_REPLICATE)
    box = dict(ddepth=cv2.CV_32F, ksize=(3, 3), normalize=False, borderType=cv2.BORDER_REPLICATE)
    sxx = cv2.boxFilter(cv2.multiply(ix, ix), **box)
    sxy = cv2.boxFilter(cv2.multiply(ix, iy), **box)
    syy = cv2.boxFilter(cv2.multiply(iy, iy), **box)
    tr = cv2.add(sxx, syy)
    det = cv2.subtract(cv2.multiply(sxx, syy), cv2.multiply(sxy, sxy))
    c = cv2.subtract(det, cv2.multiply(tr, tr, scale=kappa))
    return np.ascontiguousarray(c[2:-2, 2:-2])
