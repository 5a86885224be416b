"""Drive the reference package's own evaluator on the thesis Harris program.

TEST INFRASTRUCTURE ONLY — needs the reference package ``sges``: the tree under
``/root/reference`` (build container) or the unmodified package pip-installed into
``baseline/_ref`` (which travels to the GPU box).  Used by
``tests/golden/make_golden.py`` (which commits its outputs as fixtures), by tests
that skip when the reference is missing, and by ``bench.py --impl reference`` to time
the reference evaluator itself.

The term is the point-free spelling of the thesis Rise ``harris``
(grayscale 2430-2432, slide2d/stencil2d 2461-2465,
conv3x3 2466-2468, Sx/Sy 2470-2472, +3x3 2474, coarsity 2437-2443) in the
package's surface syntax; see SURVEY.md Appendix A for why every stencil body is
point-free (infer.py:261-292) and why -1 and the negative weights are ambient
values (parser.py:323-349 has no unary minus).  It is parsed with
``parser.parse_term`` (parser.py:352), typed with ``infer.from_named``
(infer.py:393) to ``n.m.f32`` and evaluated with ``evalref.eval_term``
(evalref.py:119) in Python f64.

The same module also exposes the in-package drop-in hook:
``harris`` as an *ambient primitive* with scheme ``3.(?n+4).(?m+4).f32 ->
?n.?m.f32`` — ``env`` entries are instantiated per use (infer.py:190-196,
252-253) and ``amb`` entries override primitive semantics (evalref.py:142-144).
"""
from __future__ import annotations

import os
import sys
from typing import Callable, Optional

import numpy as np

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _default_src() -> str:
    """HARRIS_REFERENCE_SRC, else the reference tree (build container), else the unmodified
    reference package pip-installed into baseline/_ref (travels to the GPU box; see
    __graft_entry__.build)."""
    env = os.environ.get("HARRIS_REFERENCE_SRC")
    if env:
        return env
    for cand in ("/root/reference/pkg/src", os.path.join(_ROOT, "baseline", "_ref")):
        if os.path.isdir(os.path.join(cand, "sges")):
            return cand
    return "/root/reference/pkg/src"


REFERENCE_SRC = _default_src()


def available() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "sges"))


def _sges():
    if not available():
        raise RuntimeError(f"reference package not found at {REFERENCE_SRC}")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    from sges import infer, nat, parser, types  # noqa: F401
    from sges import evalref
    return parser, types, nat, infer, evalref


def _arr(types, nat, *dims):
    t = types.scalar()
    for s in reversed(dims):
        t = types.array(nat.const(s) if isinstance(s, int) else s, t)
    return types.data(t)


GRAY = "(map (map (dot wgray)) (map transpose (transpose rgb)))"


def _nbh(i: str) -> str:
    return f"(map (map join) (map transpose (slide 3 1 (map (slide 3 1) {i}))))"


def _zip2(a: str, b: str) -> str:
    return f"(map (\\r. zip (fst r) (snd r)) (zip {a} {b}))"


def _mul2(a: str, b: str) -> str:
    return f"(map (map (\\q. mul (fst q) (snd q))) {_zip2(a, b)})"


def _sum3(i: str) -> str:
    return f"(map (map (reduce add 0)) {_nbh(i)})"


def _binom3(i: str) -> str:
    """the reference's binomial stencil (its `binomial` goal's initial form, evalref weights2d)"""
    return f"(map (map (dot (join weights2d))) {_nbh(i)})"


def harris_source(window: str = "box") -> str:
    """The thesis Harris term; window "binomial" replaces the 3x3 '+' box sums by the binomial
    filter, the variant PAPER.md:3937-3938 names ("sometimes used as part of the Harris corner
    detection instead of the 3x3 '+' convolution")."""
    IX, IY = (f"(map (map (dot (join {w}))) {_nbh(GRAY)})" for w in ("wsx", "wsy"))
    coars = (r"(\p. (\a. (\b. (\c. (\det. (\tr. add det (mul neg1 (mul (mul 0.04 tr) tr)))"
             r" (add a c)) (add (mul a c) (mul neg1 (mul b b)))) (snd (snd p))) (fst (snd p))) (fst p))")
    win = {"box": _sum3, "binomial": _binom3}[window]
    return f"map (map {coars}) {_zip2(win(_mul2(IX, IX)), _zip2(win(_mul2(IX, IY)), win(_mul2(IY, IY))))}"


WEIGHTS = {
    "wgray": [0.299, 0.587, 0.114],
    "wsx": [[-1 / 12, 0, 1 / 12], [-2 / 12, 0, 2 / 12], [-1 / 12, 0, 1 / 12]],
    "wsy": [[-1 / 12, -2 / 12, -1 / 12], [0, 0, 0], [1 / 12, 2 / 12, 1 / 12]],
    "neg1": -1.0,
}


def typed_term(window: str = "box"):
    """Parse and type the Harris term; returns (term, type_string)."""
    parser, types, nat, infer, _ = _sges()
    n, m = nat.var("n"), nat.var("m")
    env = {"rgb": _arr(types, nat, 3, nat.add(n, nat.const(4)), nat.add(m, nat.const(4))),
           "wgray": _arr(types, nat, 3), "wsx": _arr(types, nat, 3, 3),
           "wsy": _arr(types, nat, 3, 3), "neg1": types.data(types.scalar())}
    term = infer.from_named(parser.parse_term(harris_source(window)), env=env, sizes={"n", "m"})
    return term, types.show(term.ty) if hasattr(types, "show") else str(term.ty)


def harris_sges(rgb: np.ndarray, window: str = "box") -> np.ndarray:
    """Evaluate the thesis Harris program with the reference evaluator (f64).

    ``rgb``: float32 (3, H, W); the f32 values are passed exactly (as Python
    floats) so the oracle and the GPU see identical inputs."""
    rgb = np.asarray(rgb, dtype=np.float32)
    H, W = rgb.shape[1:]
    if H < 5 or W < 5:
        raise ValueError("H, W must be >= 5")
    _, _, _, _, evalref = _sges()
    term, _ = typed_term(window)
    amb = dict(WEIGHTS)
    amb["rgb"] = rgb.astype(np.float64).tolist()
    out = evalref.eval_term(term, (), amb, {"n": H - 4, "m": W - 4})
    return np.asarray(out, dtype=np.float64)


BINOMIAL_INITIAL = "map (map (dot (join weights2d))) (map (map join) (map transpose (slide 3 1 (map (slide 3 1) input))))"
BINOMIAL_SEPARATED = r"map (\l. map (dot weightsH) (slide 3 1 (map (dot weightsV) (transpose l)))) (slide 3 1 input)"


def binomial_sges(img: np.ndarray, form: str = "separated") -> np.ndarray:
    """The reference's binomial rewrite goal (Fig. binom-rewrite),
    initial (direct 2-D) or separated (vertical then horizontal) program, evaluated by
    ``evalref.eval_term`` in f64 with the reference's weights (evalref.py:112-115)."""
    parser, types, nat, infer, evalref = _sges()
    img = np.asarray(img, dtype=np.float32)
    H, W = img.shape
    n, m = nat.var("n"), nat.var("m")
    env = {"input": _arr(types, nat, nat.add(n, nat.const(2)), nat.add(m, nat.const(2)))}
    src = BINOMIAL_INITIAL if form == "initial" else BINOMIAL_SEPARATED
    term = infer.from_named(parser.parse_term(src), env=env, sizes={"n", "m"})
    out = evalref.eval_term(term, (), {"input": img.astype(np.float64).tolist()}, {"n": H - 2, "m": W - 2})
    return np.asarray(out, dtype=np.float64)


def register_ambient_harris(env: dict, amb: dict, impl: Callable[[np.ndarray], np.ndarray]):
    """Register ``harris`` as an ambient Rise primitive.

    ``impl`` maps a float32 (3, H, W) array to an (H-4, W-4) array; values cross
    the boundary as nested Python lists (evalref.py:1-7)."""
    parser, _, _, _, _ = _sges()
    env["harris"] = parser.parse_type("3.(?n+4).(?m+4).f32 -> ?n.?m.f32")

    def _call(rgb_lists):
        arr = np.asarray(rgb_lists, dtype=np.float32)
        return np.asarray(impl(arr), dtype=np.float64).tolist()

    amb["harris"] = _call
    return env, amb


def eval_via_ambient(rgb: np.ndarray, impl: Callable[[np.ndarray], np.ndarray]) -> np.ndarray:
    """Type-check and evaluate the Rise program ``harris rgb`` where ``harris`` is
    the ambient primitive backed by ``impl`` (e.g. the B200 kernel)."""
    parser, types, nat, infer, evalref = _sges()
    rgb = np.asarray(rgb, dtype=np.float32)
    H, W = rgb.shape[1:]
    env = {"rgb": _arr(types, nat, 3, H, W)}
    amb: dict = {}
    register_ambient_harris(env, amb, impl)
    term = infer.from_named(parser.parse_term("harris rgb"), env=env, sizes=set())
    amb["rgb"] = rgb.astype(np.float64).tolist()
    return np.asarray(evalref.eval_term(term, (), amb, {}), dtype=np.float64)
