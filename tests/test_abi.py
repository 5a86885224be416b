"""CPU: the C-ABI library loads and exports exactly what include/harris_b200.h declares.

No compute calls here (no GPU in the build container); the only call that
touches CUDA is harris_init, which must fail cleanly with an error code.
"""
import ctypes
import os
import re
import subprocess

import pytest
import torch

import paper_2212_12035_b200 as hb
from paper_2212_12035_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "harris_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"HARRIS_API\s+[\w\s\*]+?\b(harris_\w+)\s*\(", src)))


def test_header_declares_the_python_symbol_list():
    assert declared_symbols() == sorted(_lib.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (harris_\w+)", out))
    assert exported == set(declared_symbols())


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_tma_kernel_uses_tma_in_sass():
    out = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTMALDG" in out          # cp.async.bulk.tensor (TMA) loads
    assert "SYNCS" in out            # mbarrier transaction counting
    assert "SHFL.DOWN" in out        # warp-shuffle halo exchange


def test_abi_version_and_strerror():
    L = _lib.lib()
    assert L.harris_abi_version() == 1
    for code in range(0, -9, -1):
        s = L.harris_strerror(code)
        assert s and b"unknown" not in s
    assert b"unknown" in L.harris_strerror(-99)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU error path")
def test_init_without_gpu_is_an_error_code():
    h = ctypes.c_void_p()
    rc = _lib.lib().harris_init(ctypes.byref(h), 0)
    assert rc in (_lib.HARRIS_ERR_NO_DEVICE, _lib.HARRIS_ERR_UNSUPPORTED_DEVICE)
    assert not h.value
    with pytest.raises(hb.HarrisError):
        hb.HarrisContext(0)


def test_null_ctx_is_rejected_without_cuda():
    L = _lib.lib()
    assert L.harris_run(None, None, 8, 4, 8, None, 0.04, None) == _lib.HARRIS_ERR_INVALID_ARGUMENT
    assert L.harris_last_path(None) == _lib.PATH_NONE
    L.harris_destroy(None)


def test_algorithmic_bytes():
    # 12 B read per input pixel, 4 B written per output pixel (BASELINE.json)
    assert hb.algorithmic_bytes(8188, 8188) == 12 * 8192 * 8192 + 4 * 8188 * 8188
    assert hb.algorithmic_bytes(1076, 1916, 1024) == 1024 * (12 * 1080 * 1920 + 4 * 1076 * 1916)


def test_python_wrapper_validates_before_cuda():
    with pytest.raises((ValueError, TypeError)):
        hb.harris(torch.zeros((2, 10, 10)).cuda() if torch.cuda.is_available() else torch.zeros((4, 3, 2, 2, 2)))


def test_peer_entry_points_validate_without_a_device():
    """The fused-gather entry points reject bad arguments before touching CUDA."""
    L = _lib.lib()
    h = _lib.PeerHandle()
    assert L.harris_peer_export(None, ctypes.byref(h)) == _lib.HARRIS_ERR_INVALID_ARGUMENT
    mp, p = ctypes.c_void_p(), ctypes.c_void_p()
    assert L.harris_peer_open(0, None, ctypes.byref(mp), ctypes.byref(p)) == _lib.HARRIS_ERR_INVALID_ARGUMENT
    bad = _lib.PeerHandle()
    bad.offset = -1
    assert L.harris_peer_open(0, ctypes.byref(bad), ctypes.byref(mp), ctypes.byref(p)) == \
        _lib.HARRIS_ERR_INVALID_ARGUMENT
    assert L.harris_peer_close(0, None) == _lib.HARRIS_OK
    assert L.harris_peer_signal(None, 1, None) == _lib.HARRIS_ERR_INVALID_ARGUMENT
    assert L.harris_peer_wait(None, 0, 1, None, 0, None) == _lib.HARRIS_OK
    assert L.harris_peer_wait(None, -1, 1, None, 0, None) == _lib.HARRIS_ERR_INVALID_ARGUMENT
    assert L.harris_peer_wait(None, 2, 1, None, 0, None) == _lib.HARRIS_ERR_INVALID_ARGUMENT
    assert L.harris_run_notify(None, None, 8, 64, 4, 4, None, 8, 64, 192, 1, 0.04, 0, None, 1, None) == \
        _lib.HARRIS_ERR_INVALID_ARGUMENT


def test_peer_handle_layout_and_roundtrip():
    # harris_peer_handle: 64-byte IPC handle, int64 offset, int64 bytes, int32 device, int32 reserved
    assert ctypes.sizeof(_lib.PeerHandle) == 64 + 8 + 8 + 4 + 4
    h = _lib.PeerHandle()
    for i in range(64):
        h.ipc[i] = (7 * i) & 0xFF
    h.offset, h.bytes, h.device = 4096, 1 << 30, 3
    g = _lib.PeerHandle.from_bytes(h.to_bytes())
    assert bytes(g.ipc) == bytes(h.ipc) and (g.offset, g.bytes, g.device) == (4096, 1 << 30, 3)


def test_plain_c_host_example_without_a_device():
    """examples/harris_host.c links only the C-ABI (no CUDA headers / runtime in the app);
    without a GPU it must fail cleanly through harris_init's error code."""
    exe = os.path.join(ROOT, "examples", "harris_host")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "examples")], check=True, capture_output=True)
    if torch.cuda.is_available():
        pytest.skip("a GPU is present (tests/test_gpu_parity.py runs the example)")
    r = subprocess.run([exe, "64", "136"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 4 and "harris_init" in r.stderr


def test_library_has_no_undefined_internal_symbols():
    """Every internal (harris::) symbol the library references is defined in it: a missing
    definition would only surface as a dlopen failure on the GPU box."""
    import shutil
    import subprocess
    if not shutil.which("nm"):
        pytest.skip("nm not available")
    out = subprocess.run(["nm", "-D", "--undefined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    missing = [ln for ln in out.splitlines() if "_ZN6harris" in ln]
    assert not missing, missing
