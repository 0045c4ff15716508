"""Pins of O-EXACT (oracle/exact.py, oracle/jacobi.c) against what the paper and the
mathematics fix -- never against the oracle itself.

  * planted spectrum: Pi(Q L Q^T) = Q max(L, 0) Q^T (closed form)
  * Moreau / KKT certificate of the projection onto the self-dual PSD cone:
    P >= 0, P - A >= 0, <P, P - A> = 0 (BASELINE north_star invariants)
  * idempotence, negation identity Pi(A) = A + Pi(-A)
  * 2x2 / 3x3 closed forms and brute-force minimisation over X = L L^T
  * SPEC.md worked examples (tests/golden/spec_examples.json)
  * Jacobi eigendecomposition vs numpy.linalg.eigh (LAPACK, independent code)
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.optimize import minimize

from oracle import exact
from oracle._clib import jacobi_eig
from workloads.generators import haar_q, planted

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
U = 2.0 ** -53


def psd_by_cholesky(M, delta):
    """Membership of the PSD cone by a plain Cholesky of M + delta I."""
    try:
        np.linalg.cholesky(0.5 * (M + M.T) + delta * np.eye(M.shape[0]))
        return True
    except np.linalg.LinAlgError:
        return False


@pytest.mark.parametrize("n,p", [(5, 2), (40, 3), (120, 60), (200, 10)])
def test_planted_spectrum(n, p):
    rng = np.random.default_rng(n + p)
    lam = np.concatenate([rng.uniform(0.1, 10, p), rng.uniform(-10, -0.1, n - p)])
    Q = haar_q(rng, n)
    A = planted(Q, lam)
    Pstar = (Q * np.maximum(lam, 0)) @ Q.T
    Pi = exact.project_exact(A)
    assert np.linalg.norm(Pi - Pstar) <= 1e-12 * np.linalg.norm(A) + 10 * n * U * np.abs(lam).max()


@pytest.mark.parametrize("seed", range(6))
def test_moreau_certificate(seed):
    rng = np.random.default_rng(100 + seed)
    n = [3, 8, 17, 30, 50, 64][seed]
    M = rng.standard_normal((n, n))
    A = 0.5 * (M + M.T)
    P = exact.project_exact(A)
    d = 10 * n * U * np.linalg.norm(A)
    assert psd_by_cholesky(P, d)
    assert psd_by_cholesky(P - A, d)
    assert abs(np.sum(P * (P - A))) <= 1e-12 * np.linalg.norm(A) ** 2
    # a wrong answer fails the certificate: dropping one positive eigenpair breaks P - A >= 0
    w, V = np.linalg.eigh(A)
    Pbad = (V[:, w > 0][:, 1:] * w[w > 0][1:]) @ V[:, w > 0][:, 1:].T
    assert not psd_by_cholesky(Pbad - A, d)


def test_idempotence_and_negation():
    rng = np.random.default_rng(7)
    M = rng.standard_normal((25, 25))
    A = 0.5 * (M + M.T)
    P = exact.project_exact(A)
    assert np.linalg.norm(exact.project_exact(P) - P) <= 1e-12 * np.linalg.norm(A)
    # Pi(A) = A + Pi(-A)  (PAPER.md:317 right form applied to -A)
    assert np.linalg.norm(A + exact.project_exact(-A) - P) <= 1e-12 * np.linalg.norm(A)


def _pi_2x2_closed(a, b, c):
    """lambda+- = (a+c)/2 +- sqrt(((a-c)/2)^2 + b^2), eigenvector (b, lambda - a)."""
    h = math.sqrt(((a - c) / 2) ** 2 + b * b)
    P = np.zeros((2, 2))
    for lam in ((a + c) / 2 + h, (a + c) / 2 - h):
        if lam <= 0:
            continue
        v = np.array([b, lam - a]) if abs(b) > 0 else (np.array([1.0, 0.0]) if abs(lam - a) <= abs(lam - c) else np.array([0.0, 1.0]))
        v = v / np.linalg.norm(v)
        P += lam * np.outer(v, v)
    return P


def _brute(A, starts=60, seed=0):
    """min ||A - L L^T||_F over lower-triangular L (n(n+1)/2 parameters), Nelder-Mead."""
    n = A.shape[0]
    il = np.tril_indices(n)
    rng = np.random.default_rng(seed)

    def f(x):
        L = np.zeros((n, n))
        L[il] = x
        return np.sum((A - L @ L.T) ** 2)

    best = None
    for _ in range(starts):
        r = minimize(f, rng.standard_normal(len(il[0])), method="Nelder-Mead",
                     options=dict(xatol=1e-12, fatol=1e-16, maxiter=20000, maxfev=40000))
        if best is None or r.fun < best.fun:
            best = r
    L = np.zeros((n, n))
    L[il] = best.x
    return L @ L.T


@pytest.mark.parametrize("abc", [(1.0, 0.5, 2.0), (1.0, 2.0, -1.0), (-1.0, 0.3, -2.0), (3.0, -1.5, 0.5), (0.0, 1.0, 0.0)])
def test_2x2_closed_form_and_brute_force(abc):
    a, b, c = abc
    A = np.array([[a, b], [b, c]])
    P = exact.project_exact(A)
    assert np.abs(P - _pi_2x2_closed(a, b, c)).max() <= 1e-10
    assert np.abs(P - _brute(A, starts=20)).max() <= 1e-5


def _eig3_trig(A):
    """Eigenvalues of a symmetric 3x3 by the trigonometric solution of the characteristic cubic."""
    q = np.trace(A) / 3
    B = A - q * np.eye(3)
    p = math.sqrt(np.sum(B * B) / 6)
    if p == 0:
        return np.array([q, q, q])
    r = np.linalg.det(B / p) / 2
    phi = math.acos(min(1.0, max(-1.0, r))) / 3
    l1 = q + 2 * p * math.cos(phi)
    l3 = q + 2 * p * math.cos(phi + 2 * math.pi / 3)
    return np.array([l1, 3 * q - l1 - l3, l3])


def _vec3(A, lam):
    M = A - lam * np.eye(3)
    cands = [np.cross(M[0], M[1]), np.cross(M[0], M[2]), np.cross(M[1], M[2])]
    v = max(cands, key=np.linalg.norm)
    return v / np.linalg.norm(v)


@pytest.mark.parametrize("seed", range(4))
def test_3x3_closed_form_and_brute_force(seed):
    rng = np.random.default_rng(30 + seed)
    M = rng.standard_normal((3, 3))
    A = 0.5 * (M + M.T)
    lams = _eig3_trig(A)
    Pc = sum(l * np.outer(_vec3(A, l), _vec3(A, l)) for l in lams if l > 0)
    P = exact.project_exact(A)
    assert np.abs(P - Pc).max() <= 1e-9
    if seed < 2:
        assert np.abs(P - _brute(A, starts=25, seed=seed)).max() <= 1e-4


@pytest.mark.parametrize("case", GOLD["projection"], ids=lambda c: c["cite"][:24])
def test_spec_projection_examples(case):
    A = np.array(case["A"], dtype=float)
    P, parts = exact.project_exact(A, return_parts=True)
    assert np.array_equal(np.round(P, 14) + 0.0, np.array(case["Pi"], dtype=float))
    pos, neg = exact.sign_counts(parts["w"], np.linalg.norm(A))
    assert (pos, neg) == (case["pos"], case["neg"])


@pytest.mark.parametrize("case", GOLD["eig"], ids=lambda c: c["cite"][:24])
def test_spec_eig_examples(case):
    A = np.array(case["A"], dtype=float)
    w, V, _ = jacobi_eig(A)
    assert np.array_equal(w, np.array(case["values"], dtype=float))
    assert np.array_equal(np.abs(V), np.abs(V).round())  # permuted identity columns


def test_special_cases():
    assert exact.project_exact(np.array([[-2.5]]))[0, 0] == 0.0
    assert exact.project_exact(np.array([[3.25]]))[0, 0] == 3.25
    assert np.array_equal(exact.project_exact(-np.eye(6)), np.zeros((6, 6)))
    rng = np.random.default_rng(1)
    G = rng.standard_normal((9, 9))
    S = G @ G.T  # PSD input unchanged
    assert np.linalg.norm(exact.project_exact(S) - S) <= 1e-10 * np.linalg.norm(S)


def test_sampled_optimality():
    """||Pi(A) - A|| <= ||X - A|| for 100 random PSD X (n = 12)."""
    rng = np.random.default_rng(12)
    M = rng.standard_normal((12, 12))
    A = 0.5 * (M + M.T)
    d0 = np.linalg.norm(exact.project_exact(A) - A)
    for _ in range(100):
        G = rng.standard_normal((12, rng.integers(1, 13)))
        assert d0 <= np.linalg.norm(G @ G.T * rng.uniform(0.01, 2) - A) + 1e-12


@pytest.mark.parametrize("n", [1, 2, 9, 60, 150])
def test_jacobi_vs_lapack(n):
    rng = np.random.default_rng(n)
    M = rng.standard_normal((n, n))
    A = 0.5 * (M + M.T)
    w, V, sweeps = jacobi_eig(A)
    assert sweeps > 0
    ref = np.linalg.eigvalsh(A)
    assert np.abs(w - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max()) * max(1, n / 10)
    assert np.linalg.norm(V.T @ V - np.eye(n)) <= 1e-12 * max(n, 1)
    assert np.linalg.norm((V * w) @ V.T - A) <= 1e-12 * np.linalg.norm(A) * max(1, n / 10)
    assert np.all(np.diff(w) >= 0)


def test_jacobi_rejects_nonfinite():
    A = np.eye(3)
    A[1, 2] = A[2, 1] = np.nan
    with pytest.raises(FloatingPointError):
        jacobi_eig(A)
