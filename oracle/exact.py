"""O-EXACT: the PSD-cone projection by its definition (TEST INFRASTRUCTURE; see oracle/__init__.py).

PAPER.md:308-318 (Eq. admm:eqn:eigendecomposition / admm:eqn:projection), readings R1-R4:
  Pi(A) = argmin_{X >= 0} ||A - X||_F = V+ L+ V+^T = A - V- L- V-^T,
with A = [V+ V-] diag(L+, L-) [V+ V-]^T from a full eigendecomposition (cyclic Jacobi,
oracle/jacobi.c). Eigenvalues exactly 0 contribute nothing to either form (R3).
"""
import numpy as np

from ._clib import jacobi_eig

U = 2.0 ** -53


def eig(A):
    """Full eigendecomposition by cyclic Jacobi: (w ascending, V)."""
    w, V, _ = jacobi_eig(A)
    return w, V


def project_exact(A, return_parts=False):
    """Pi(A) via Jacobi. Both closed forms are evaluated and must agree to
    10 n u ||A||_F (self-check of the two sides); Pi+ is returned, symmetrised (R24)."""
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    w, V = eig(A)
    pos = w > 0
    neg = w < 0
    Vp = V[:, pos]
    Vn = V[:, neg]
    pi_plus = (Vp * w[pos]) @ Vp.T
    pi_minus = A - (Vn * w[neg]) @ Vn.T
    pi_plus = 0.5 * (pi_plus + pi_plus.T)
    pi_minus = 0.5 * (pi_minus + pi_minus.T)
    fro = np.linalg.norm(A)
    gap = np.linalg.norm(pi_plus - pi_minus)
    if gap > 10 * max(n, 1) * U * max(fro, 1e-300) + 1e-300:
        raise AssertionError(f"closed forms disagree: {gap} vs {10 * n * U * fro}")
    if return_parts:
        return pi_plus, dict(w=w, V=V, pi_minus=pi_minus)
    return pi_plus


def sign_counts(w, fro):
    """Counts of positive / negative eigenvalues with the zero band
    |lambda| <= 1e-9 (1 + ||A||_F) counted as neither (reading R19)."""
    z = 1e-9 * (1.0 + fro)
    return int(np.sum(w > z)), int(np.sum(w < -z))
