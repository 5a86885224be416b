"""B200-native fused Harris corner detection (the data-parallel hot path of
arXiv 2212.12035).

Public API
----------
``harris(rgb, kappa=0.04)``   Rise ``harris : 3.(n+4).(m+4).f32 -> n.m.f32``
                                on CUDA or host tensors.
``HarrisContext`` / ``context``  the C-ABI context (``harris_init``/``_destroy``).
``synth_``                      device synthetic-image generator.
``shard``                       multi-GPU row-band / image sharding driver.
``sges_bridge``                 registers ``harris`` as an ambient Rise primitive
                               in the reference ``sges`` evaluator.

The compute path is ``libharris_b200.so`` (``csrc/``, sm_100a only).  There is
no CPU fallback: without the library or a B200 every entry point raises.
"""
from ._lib import HarrisError, build  # noqa: F401
from .harris import (GROUPINGS, KAPPA, HarrisContext, algorithmic_bytes, context, grouping_hbm_bytes,  # noqa: F401
                     harris, harris_frames, harris_grouping, harris_u8, stencil3x3_sep, synth_)

__version__ = "0.1.0"
