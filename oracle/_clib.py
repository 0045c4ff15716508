"""ctypes loader for oracle/jacobi.c (TEST INFRASTRUCTURE; see oracle/__init__.py).

The shared object is built by __graft_entry__.build() (or on first use here) with plain
gcc; it never links anything from paper_1912_02767_b200/.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "jacobi.c")
_SO = os.path.join(_HERE, "_liboracle.so")
_lib = None


def build(force=False):
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        dp = ctypes.POINTER(ctypes.c_double)
        L.oracle_jacobi_eig.argtypes = [ctypes.c_int, dp, ctypes.c_int, dp, dp, ctypes.c_int]
        L.oracle_jacobi_eig.restype = ctypes.c_int
        L.oracle_cholesky.argtypes = [ctypes.c_int, dp, ctypes.c_int, dp, ctypes.c_double]
        L.oracle_cholesky.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def jacobi_eig(A, max_sweeps=60):
    """Cyclic Jacobi eigendecomposition (jacobi.c). Returns (w ascending, V, sweeps)."""
    A = np.asfortranarray(np.asarray(A, dtype=np.float64))
    n = A.shape[0]
    assert A.shape == (n, n)
    w = np.zeros(n)
    V = np.zeros((n, n), order="F")
    rc = lib().oracle_jacobi_eig(n, _ptr(A), max(n, 1), _ptr(w), _ptr(V), max_sweeps)
    if rc == -3:
        raise FloatingPointError("non-finite input to jacobi_eig")
    if rc < 0:
        raise RuntimeError(f"jacobi_eig failed rc={rc}")
    return w, V, rc


def cholesky(G, pivot_floor=0.0):
    """Plain Cholesky (jacobi.c). Returns (L lower, 0) or (None, failing pivot index+1)."""
    G = np.asfortranarray(np.asarray(G, dtype=np.float64))
    n = G.shape[0]
    L = np.zeros((n, n), order="F")
    rc = lib().oracle_cholesky(n, _ptr(G), max(n, 1), _ptr(L), float(pivot_floor))
    return (L if rc == 0 else None), rc
