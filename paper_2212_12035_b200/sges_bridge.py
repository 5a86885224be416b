"""Register the fused B200 kernel as an ambient Rise primitive in the reference
``sges`` package (the in-package drop-in hook of SURVEY.md §8b(ii)).

The reference's type checker treats any name in ``env`` as a polymorphic scheme
instantiated per use (infer.py:190-196, 252-253) and its evaluator lets ``amb``
override primitive semantics (evalref.py:142-144).  Registering

    env["harris"] = 3.(?n+4).(?m+4).f32 -> ?n.?m.f32
    amb["harris"] = <callable running the fused kernel>

makes ``harris rgb`` type-check to ``n.m.f32`` and evaluate on the GPU.  Values
cross that boundary as nested Python lists (evalref.py:1-7), so this bridge is
for interoperability and parity harnesses, not for throughput.

The reference type checker does not reject degenerate sizes (it solves
``?m = -2`` for a 3x5x2 input, nat.py:211-239), so the bridge validates
``H, W >= 5`` itself before calling the C-ABI (which also rejects them).
"""
from __future__ import annotations

import os
import sys
from typing import Callable, Optional

import numpy as np

HARRIS_SCHEME = "3.(?n+4).(?m+4).f32 -> ?n.?m.f32"


_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sges(reference_src: Optional[str] = None):
    src = reference_src or os.environ.get("HARRIS_REFERENCE_SRC")
    if not src and os.path.isdir(os.path.join(_ROOT, "baseline", "_ref", "sges")):
        src = os.path.join(_ROOT, "baseline", "_ref")  # the pip-installed reference (__graft_entry__.build)
    if src and src not in sys.path:
        sys.path.insert(0, src)
    try:
        from sges import parser  # noqa: F401
    except ImportError as e:  # pragma: no cover - depends on the user's install
        raise ImportError("the reference package `sges` is not importable; set HARRIS_REFERENCE_SRC "
                          "to its src directory") from e
    from sges import evalref, infer, parser
    return parser, infer, evalref


def gpu_impl(kappa: float = 0.04, window: str = "box") -> Callable[[np.ndarray], np.ndarray]:
    """(3, H, W) float32 host array -> (H-4, W-4) through the fused kernel."""
    import torch

    from .harris import harris

    def run(rgb: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(np.ascontiguousarray(rgb, dtype=np.float32)).cuda()
        out = harris(t, kappa, window=window)
        return out.cpu().numpy()

    return run


def register(env: dict, amb: dict, impl: Optional[Callable[[np.ndarray], np.ndarray]] = None,
             reference_src: Optional[str] = None, name: str = "harris", window: str = "box") -> tuple[dict, dict]:
    """Add the ``harris`` scheme to a type environment and its implementation to
    an evaluator ambient map; ``impl`` defaults to the B200 kernel.  ``window="binomial"``
    (registered e.g. as ``name="harris_binomial"``) is the Harris variant with the binomial
    window, the sges program ``oracle/sges_oracle.harris_source("binomial")``."""
    parser, _, _ = _sges(reference_src)
    fn = impl or gpu_impl(window=window)
    env[name] = parser.parse_type(HARRIS_SCHEME)

    def _call(rgb_lists):
        arr = np.asarray(rgb_lists, dtype=np.float32)
        if arr.ndim != 3 or arr.shape[0] != 3 or arr.shape[1] < 5 or arr.shape[2] < 5:
            raise ValueError(f"harris needs a 3 x (n+4) x (m+4) input with n, m >= 1, got {arr.shape}")
        return np.asarray(fn(arr), dtype=np.float64).tolist()

    amb[name] = _call
    return env, amb


BINOMIAL_SCHEME = "(?n+2).(?m+2).f32 -> ?n.?m.f32"


def gpu_binomial_impl() -> Callable[[np.ndarray], np.ndarray]:
    import torch

    from .harris import stencil3x3_sep

    def run(img: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)).cuda()
        return stencil3x3_sep(t).cpu().numpy()

    return run


def register_binomial(env: dict, amb: dict, impl: Optional[Callable[[np.ndarray], np.ndarray]] = None,
                      reference_src: Optional[str] = None) -> tuple[dict, dict]:
    """Register ``binomial`` (the reference's separated binomial goal as one primitive,
    PAPER.md:3935-4016) with scheme ``(?n+2).(?m+2).f32 -> ?n.?m.f32``; ``impl`` defaults
    to the separable-stencil kernel on the B200."""
    parser, _, _ = _sges(reference_src)
    fn = impl or gpu_binomial_impl()
    env["binomial"] = parser.parse_type(BINOMIAL_SCHEME)

    def _call(img_lists):
        arr = np.asarray(img_lists, dtype=np.float32)
        if arr.ndim != 2 or arr.shape[0] < 3 or arr.shape[1] < 3:
            raise ValueError(f"binomial needs an (n+2) x (m+2) input with n, m >= 1, got {arr.shape}")
        return np.asarray(fn(arr), dtype=np.float64).tolist()

    amb["binomial"] = _call
    return env, amb


def evaluate(src: str, env: dict, amb: dict, sizes=(), nenv: Optional[dict] = None,
             reference_src: Optional[str] = None):
    """Parse, type and evaluate a Rise program that may call ``harris``."""
    parser, infer, evalref = _sges(reference_src)
    term = infer.from_named(parser.parse_term(src), env=env, sizes=set(sizes))
    return term, evalref.eval_term(term, (), amb, nenv or {})
