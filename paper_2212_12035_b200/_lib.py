"""ctypes binding of ``libharris_b200.so`` (the C-ABI in ``include/harris_b200.h``).

The library is built in-tree by ``build()`` (``make -C csrc``) and travels with
the repo snapshot.  There is no fallback: if the library is missing or cannot be
loaded, :func:`lib` raises, and on a machine without a B200 ``harris_init``
fails with ``HARRIS_ERR_NO_DEVICE`` / ``HARRIS_ERR_UNSUPPORTED_DEVICE``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HARRIS_LIB") or os.path.join(PKG_DIR, "libharris_b200.so")  # HARRIS_LIB: dev A/B only
CSRC = os.path.join(PKG_DIR, "csrc")

HARRIS_OK = 0
HARRIS_ERR_INVALID_ARGUMENT = -1
HARRIS_ERR_SIZE = -2
HARRIS_ERR_ALIGNMENT = -3
HARRIS_ERR_CUDA = -4
HARRIS_ERR_NO_DEVICE = -5
HARRIS_ERR_TMA = -6
HARRIS_ERR_OUT_OF_MEMORY = -7
HARRIS_ERR_UNSUPPORTED_DEVICE = -8

FLAG_EXACT_ORDER = 0x1
FLAG_FORCE_GENERIC = 0x2
FLAG_FORCE_TMA = 0x4
FLAG_PDL = 0x8
FLAG_PDL_INDEPENDENT = 0x10
FLAG_BINOMIAL_WINDOW = 0x20

PATH_NONE, PATH_TMA, PATH_GENERIC, PATH_LDG, PATH_PAIR, PATH_QUAD = 0, 1, 2, 3, 4, 5

# every symbol include/harris_b200.h declares (checked by tests/test_abi.py)
EXPORTED_SYMBOLS = (
    "harris_init", "harris_init_ex", "harris_options_default", "harris_destroy", "harris_run", "harris_run_batched", "harris_run_strided",
    "harris_run_host", "harris_run_frames", "harris_run_frames_u8", "harris_synth_fill", "harris_plan", "harris_last_path", "harris_device",
    "harris_num_sms", "harris_strerror", "harris_last_cuda_error", "harris_abi_version",
    "harris_grouping_scratch_bytes", "harris_grouping_launches", "harris_run_grouping",
    "harris_run_u8", "harris_run_host_u8", "harris_stencil3x3_sep",
    "harris_peer_export", "harris_peer_open", "harris_peer_close", "harris_run_notify",
    "harris_peer_signal", "harris_peer_wait",
)

L2_EVICT_FIRST, L2_EVICT_NORMAL, L2_EVICT_LAST = 0, 1, 2

GROUPING_UNFUSED, GROUPING_SOBEL_PROD, GROUPING_SOBEL, GROUPING_FUSED = 1, 2, 3, 4


class HarrisError(RuntimeError):
    def __init__(self, code: int, where: str, detail: str = ""):
        self.code = code
        msg = f"{where}: {strerror(code)} ({code})"
        if detail:
            msg += f": {detail}"
        super().__init__(msg)


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("path", ctypes.c_int32), ("warps_per_cta", ctypes.c_int32), ("stages", ctypes.c_int32),
        ("rows_per_stage", ctypes.c_int32), ("band_rows", ctypes.c_int64), ("bands", ctypes.c_int64),
        ("col_segments", ctypes.c_int64), ("tiles", ctypes.c_int64), ("grid_ctas", ctypes.c_int64),
        ("smem_bytes", ctypes.c_int64), ("groups", ctypes.c_int32), ("tma_config", ctypes.c_int32),
        ("strip_cols", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


class Options(ctypes.Structure):
    """harris_options (include/harris_b200.h): fill with harris_options_default first."""
    _fields_ = [("struct_size", ctypes.c_uint32), ("l2_policy", ctypes.c_int32), ("band_rows", ctypes.c_int32),
                ("pdl", ctypes.c_int32), ("reserved", ctypes.c_int32 * 4)]


class PeerHandle(ctypes.Structure):
    """harris_peer_handle: a CUDA IPC handle plus the pointer's offset in its allocation."""
    _fields_ = [("ipc", ctypes.c_ubyte * 64), ("offset", ctypes.c_int64), ("bytes", ctypes.c_int64),
                ("device", ctypes.c_int32), ("reserved", ctypes.c_int32)]

    def to_bytes(self) -> bytes:
        return bytes(ctypes.string_at(ctypes.addressof(self), ctypes.sizeof(self)))

    @classmethod
    def from_bytes(cls, b: bytes) -> "PeerHandle":
        if len(b) != ctypes.sizeof(cls):
            raise ValueError("bad harris_peer_handle size")
        h = cls()
        ctypes.memmove(ctypes.addressof(h), b, len(b))
        return h


_lib = None


def build(force: bool = False) -> str:
    """Compile the CUDA library for sm_100a in-tree (nvcc cross-compiles without a GPU)."""
    args = ["make", "-C", CSRC] + (["-B"] if force else [])
    subprocess.run(args, check=True, stdout=subprocess.DEVNULL)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C {CSRC}); "
                           "there is no non-CUDA fallback")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, u32, u64, f32 = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint32,
                                   ctypes.c_uint64, ctypes.c_float)
    sig = {
        "harris_init": ([ctypes.POINTER(vp), i32], i32),
        "harris_init_ex": ([ctypes.POINTER(vp), i32, ctypes.POINTER(Options)], i32),
        "harris_options_default": ([ctypes.POINTER(Options)], None),
        "harris_destroy": ([vp], None),
        "harris_run": ([vp, vp, i64, i64, i64, vp, f32, vp], i32),
        "harris_run_batched": ([vp, vp, i64, i64, vp, i64, f32, vp], i32),
        "harris_run_strided": ([vp, vp, i64, i64, i64, i64, vp, i64, i64, i64, i64, f32, u32, vp], i32),
        "harris_run_host": ([vp, vp, i64, i64, i64, vp, i64, f32, u32], i32),
        "harris_run_frames": ([vp, ctypes.POINTER(vp), i64, i64, i64, ctypes.POINTER(vp), i64, i64, i64, f32, u32, vp],
                              i32),
        "harris_run_frames_u8": ([vp, ctypes.POINTER(vp), i64, i64, i64, ctypes.POINTER(vp), i64, i64, f32, u32, vp],
                                 i32),
        "harris_synth_fill": ([vp, i64, i64, i64, i64, i64, i64, i64, i64, u64, i32, vp], i32),
        "harris_plan": ([vp, i64, i64, i64, vp, i64, i64, i64, vp, i64, i64, u32, ctypes.POINTER(PlanInfo)], i32),
        "harris_last_path": ([vp], i32),
        "harris_device": ([vp], i32),
        "harris_num_sms": ([vp], i32),
        "harris_strerror": ([i32], ctypes.c_char_p),
        "harris_last_cuda_error": ([vp], ctypes.c_char_p),
        "harris_abi_version": ([], i32),
        "harris_grouping_scratch_bytes": ([i32, i64, i64], i64),
        "harris_grouping_launches": ([i32], i32),
        "harris_run_grouping": ([vp, i32, vp, i64, i64, vp, vp, i64, f32, u32, vp], i32),
        "harris_run_u8": ([vp, vp, i64, i64, i64, i64, vp, i64, i64, i64, f32, u32, vp], i32),
        "harris_run_host_u8": ([vp, vp, i64, i64, i64, vp, i64, f32, u32], i32),
        "harris_stencil3x3_sep": ([vp, vp, i64, i64, i64, i64, vp, i64, i64, i64, ctypes.POINTER(f32),
                                   ctypes.POINTER(f32), u32, vp], i32),
        "harris_peer_export": ([vp, ctypes.POINTER(PeerHandle)], i32),
        "harris_peer_open": ([i32, ctypes.POINTER(PeerHandle), ctypes.POINTER(vp), ctypes.POINTER(vp)], i32),
        "harris_peer_close": ([i32, vp], i32),
        "harris_run_notify": ([vp, vp, i64, i64, i64, i64, vp, i64, i64, i64, i64, f32, u32, vp, u32, vp], i32),
        "harris_peer_signal": ([vp, u32, vp], i32),
        "harris_peer_wait": ([vp, i32, u32, vp, i64, vp], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def strerror(code: int) -> str:
    try:
        return lib().harris_strerror(code).decode()
    except Exception:  # pragma: no cover - library missing
        return f"harris error {code}"


def check(code: int, where: str, ctx=None) -> None:
    if code != HARRIS_OK:
        detail = ""
        if ctx is not None:
            try:
                detail = lib().harris_last_cuda_error(ctx).decode()
            except Exception:  # pragma: no cover
                detail = ""
        raise HarrisError(code, where, detail)
