"""Pins of O-LOBPCG (oracle/lobpcg.py): Rayleigh-Ritz (Alg. 2), Cholesky-QR, LOBPCG (Alg. 3),
the side rule and Theorem 3 -- each against a definition,
a closed form, an invariant or LAPACK (numpy), never against the oracle itself."""
import json
import os

import numpy as np
import pytest

from oracle import lobpcg as L
from oracle.philox import gaussian_block
from workloads.generators import haar_q, planted

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _rand_sym(n, seed):
    M = np.random.default_rng(seed).standard_normal((n, n))
    return 0.5 * (M + M.T)


# ----------------------------------------------------------------- Cholesky-QR
def test_cholesky_qr_orthonormal_input_is_identity_up_to_sign():
    Q0, _ = np.linalg.qr(np.random.default_rng(1).standard_normal((20, 5)))
    Q, _ = L.cholesky_qr(Q0)
    assert np.abs(np.abs(Q) - np.abs(Q0)).max() < 1e-12


def test_cholesky_qr_rank_deficient_signal():
    e1 = np.zeros((6, 1))
    e1[0] = 1
    with pytest.raises(L.RankDeficient):
        L.cholesky_qr(np.hstack([e1, e1]))
    # the paper's fallback (Householder QR) drops the dependent column
    Q = L.orthonormalize(np.hstack([e1, e1]))
    assert Q.shape[1] == 1


def test_cholesky_qr_random_span():
    S = np.random.default_rng(2).standard_normal((20, 5))
    Q, _ = L.cholesky_qr(S)
    assert np.linalg.norm(Q.T @ Q - np.eye(5)) <= 1e-12
    # same span: projecting S onto span(Q) reproduces S (Householder QR of numpy as span oracle)
    Qh, _ = np.linalg.qr(S)
    assert np.linalg.norm(Q @ (Q.T @ S) - S) <= 1e-10
    assert np.linalg.norm(Qh @ (Qh.T @ Q) - Q) <= 1e-10


# ----------------------------------------------------------------- Rayleigh-Ritz
@pytest.mark.parametrize("case", GOLD["rayleigh_ritz"], ids=lambda c: c["cite"][:20])
def test_rr_spec_examples(case):
    A = np.array(case["A"], dtype=float)
    S = np.array(case["S"], dtype=float)
    V, w = L.rayleigh_ritz(A, S)
    assert np.allclose(w, case["values"], atol=1e-14)
    assert np.allclose(L.residual_norms(A, V, w), case["resid"], atol=1e-14)


def test_rr_random_consistency():
    A = _rand_sym(8, 3)
    S = np.random.default_rng(4).standard_normal((8, 3))
    V, w = L.rayleigh_ritz(A, S)
    assert np.linalg.norm(V.T @ A @ V - np.diag(w)) <= 1e-12  # Theorem 3 hypothesis
    Qs, _ = np.linalg.qr(S)
    assert np.linalg.norm(Qs @ (Qs.T @ V) - V) <= 1e-12  # Ritz vectors lie in span(S)
    assert np.all(np.diff(w) >= 0)  # Alg. 2 orders ascending


def test_rr_minimises_residual_over_rotations():
    """Ritz pairs minimise ||A V - V M||_F over orthonormal bases of span(S)."""
    A = _rand_sym(12, 5)
    S = np.random.default_rng(6).standard_normal((12, 4))
    V, w = L.rayleigh_ritz(A, S)
    best = np.linalg.norm(A @ V - V * w)
    rng = np.random.default_rng(7)
    for _ in range(50):
        Z, _ = np.linalg.qr(rng.standard_normal((4, 4)))
        W = V @ Z
        M = np.diag(np.diag(W.T @ A @ W))
        assert best <= np.linalg.norm(A @ W - W @ M) + 1e-12


def test_residual_spec_example():
    c = GOLD["residual"][0]
    A = np.array(c["A"], dtype=float)
    r = L.residual_norms(A, np.array(c["v"], dtype=float)[:, None], np.array([c["lam"]], dtype=float))
    assert r[0] == c["resid"]


# ----------------------------------------------------------------- LOBPCG
def test_lobpcg_diag_single_positive():
    c = GOLD["lobpcg"][0]
    B = np.diag(np.array(c["diag"], dtype=float))
    X0 = np.random.default_rng(1).standard_normal((5, 1))
    res = L.lobpcg_pos(B, X0, 1e-10, max_iter=200, cold=True)
    pos = res.theta > 0
    assert res.status == L.OK
    assert np.allclose(res.theta[pos], c["values"], atol=1e-10)
    v = res.X[:, pos][:, 0]
    assert abs(abs(v[4]) - 1) < 1e-10


def test_lobpcg_negative_definite():
    c = GOLD["lobpcg"][1]
    B = np.diag(np.array(c["diag"], dtype=float))
    res = L.lobpcg_pos(B, np.random.default_rng(2).standard_normal((4, 1)), 1e-10, cold=True)
    assert res.status == L.OK
    assert int(np.sum(res.theta > 0)) == 0


def test_lobpcg_planted_three_positive():
    """{2,3,4} among 27 values in [-10,-1] (Q L Q^T)."""
    rng = np.random.default_rng(3)
    lam = np.concatenate([[2.0, 3.0, 4.0], rng.uniform(-10, -1, 27)])
    Q = haar_q(rng, 30)
    B = planted(Q, lam)
    res = L.lobpcg_pos(B, gaussian_block(30, 5, 1, 0), 1e-9, cold=True)
    pos = res.theta > 0
    assert res.status == L.OK
    assert np.allclose(np.sort(res.theta[pos]), [2.0, 3.0, 4.0], atol=1e-9)


@pytest.mark.parametrize("seed", range(8))
def test_ritz_count_and_monotone_largest(seed):
    """Positive Ritz count <= true positive count (Cauchy interlacing) and the
    largest Ritz value is non-decreasing, at every iteration (max_iter = k)."""
    n = 40
    A = _rand_sym(n, 50 + seed) - 0.8 * np.eye(n)
    true_pos = int(np.sum(np.linalg.eigvalsh(A) > 1e-9 * (1 + np.linalg.norm(A))))
    X0 = gaussian_block(n, 6, seed, 0)
    last = -np.inf
    for k in range(0, 12):
        res = L.lobpcg_pos(A, X0, 1e-12, max_iter=k, cold=True, locking="soft")
        assert int(np.sum(res.theta > 0)) <= true_pos
        assert res.theta[0] >= last - 1e-12
        last = res.theta[0]


@pytest.mark.parametrize("locking", ["soft", "hard"])
def test_converged_values_within_residual_bounds(locking):
    """Kato-Temple / Weyl: |theta - lambda| <= min(r, r^2/gap) + rounding (SPEC.md:553 #7)."""
    rng = np.random.default_rng(9)
    lam = np.concatenate([rng.uniform(0.5, 5, 6), rng.uniform(-5, -0.5, 54)])
    Q = haar_q(rng, 60)
    A = planted(Q, lam)
    res = L.lobpcg_pos(A, gaussian_block(60, 8, 2, 0), 1e-6, cold=True, locking=locking)
    assert res.status == L.OK
    pos = res.theta > 0
    th = np.sort(res.theta[pos])[::-1]
    ref = np.sort(lam[lam > 0])[::-1]
    assert len(th) == len(ref)
    r = res.r[pos][np.argsort(-res.theta[pos])]
    gaps = np.array([np.min(np.abs(np.delete(lam, np.argmin(np.abs(lam - t))) - t)) for t in th])
    assert np.all(np.abs(th - ref) <= np.minimum(r, r ** 2 / gaps) + 1e-12)


def test_warm_start_beats_cold():
    """resuming on a perturbed matrix converges in fewer iterations than a cold start
    (median over 20 seeds)."""
    warm_it, cold_it = [], []
    for seed in range(20):
        rng = np.random.default_rng(200 + seed)
        n = 50
        lam = np.concatenate([rng.uniform(0.1, 5, 5), rng.uniform(-5, -0.1, 45)])
        Q = haar_q(rng, n)
        A0 = planted(Q, lam)
        G = rng.standard_normal((n, n))
        A1 = A0 + 1e-3 * 0.5 * (G + G.T)
        r0 = L.lobpcg_pos(A0, gaussian_block(n, 7, seed, 0), 1e-8, cold=True)
        warm = L.lobpcg_pos(A1, r0.X, 1e-8)
        cold = L.lobpcg_pos(A1, gaussian_block(n, 7, seed, 1), 1e-8, cold=True)
        warm_it.append(warm.iters)
        cold_it.append(cold.iters)
    assert np.median(warm_it) < np.median(cold_it)


def test_expansion_finds_all_positives():
    """A block narrower than the positive count must expand."""
    rng = np.random.default_rng(11)
    n = 90
    lam = np.concatenate([rng.uniform(0.5, 3, 12), rng.uniform(-3, -0.5, n - 12)])
    Q = haar_q(rng, n)
    A = planted(Q, lam)
    res = L.lobpcg_pos(A, gaussian_block(n, 4, 1, 0), 1e-9, q=5, cold=True)
    assert res.expansions >= 2
    assert res.status == L.OK
    assert np.allclose(np.sort(res.theta[res.theta > 0]), np.sort(lam[lam > 0]), atol=1e-8)


# ----------------------------------------------------------------- Theorem 3
def _perp_term(A, V):
    """||Pi(V_perp^T A V_perp)||_F by an independent full eigendecomposition (LAPACK)."""
    n, k = V.shape
    Qf, _ = np.linalg.qr(np.hstack([V, np.random.default_rng(0).standard_normal((n, n - k))]))
    Vp = Qf[:, k:]
    w = np.linalg.eigvalsh(Vp.T @ A @ Vp)
    return float(np.sqrt(np.sum(np.maximum(w, 0) ** 2)))


@pytest.mark.parametrize("n", [10, 20, 40])
@pytest.mark.parametrize("tol", [1e-1, 1e-3, 1e-6])
def test_theorem3_with_exact_perp(n, tol):
    """2||R||^2 + ||Pi(V_perp^T A V_perp)||^2 >= ||V L V^T - Pi(A)||^2 for any Rayleigh-Ritz
    output: here LOBPCG stopped early (max_iter 0..3) so R is far from zero. 0 violations."""
    viol = 0
    for seed in range(8):
        A = _rand_sym(n, 1000 * n + seed)
        w, Vf = np.linalg.eigh(A)
        Pstar = (Vf[:, w > 0] * w[w > 0]) @ Vf[:, w > 0].T
        for k in range(4):
            res = L.lobpcg_pos(A, gaussian_block(n, max(2, n // 5), seed, k), tol, max_iter=k, cold=True)
            pos = res.theta > 0
            V, th = res.X[:, pos], res.theta[pos]
            R = A @ V - V * th
            lhs = np.linalg.norm((V * th) @ V.T - Pstar) ** 2
            rhs = 2 * np.sum(R * R) + _perp_term(A, V) ** 2
            if lhs > rhs * (1 + 1e-10) + 1e-24:
                viol += 1
    assert viol == 0


def test_reported_bound_dominates_when_perp_zero():
    """Reported eps (perp term 0) >= true error whenever no positive eigenvalue is
    missed (positive counts match)."""
    checked = 0
    for seed in range(12):
        rng = np.random.default_rng(500 + seed)
        n = 60
        p = int(rng.integers(2, 10))
        lam = np.concatenate([rng.uniform(0.01, 3, p), rng.uniform(-3, -0.01, n - p)])
        Q = haar_q(rng, n)
        A = planted(Q, lam)
        Pstar = (Q * np.maximum(lam, 0)) @ Q.T
        for tol in (1e-2, 1e-5, 1e-9):
            res = L.lobpcg_pos(A, gaussian_block(n, 12, seed, 0), tol, cold=True)
            pos = res.theta > 0
            if int(pos.sum()) != p:
                continue
            V, th = res.X[:, pos], res.theta[pos]
            err = np.linalg.norm((V * th) @ V.T - Pstar)
            assert L.error_bound(A, res.X, res.theta) >= err
            checked += 1
    assert checked >= 20


# ----------------------------------------------------------------- side rule
@pytest.mark.parametrize("case", GOLD["select_mode"], ids=lambda c: c["cite"][:20])
def test_select_mode(case):
    ctx = L.Context(case["n"])
    ctx.last_pos, ctx.last_neg = case["pos"], case["neg"]
    assert ctx.select_mode() == case["mode"]


def test_select_mode_cold_and_ties():
    ctx = L.Context(30)
    assert ctx.select_mode() == L.POS  # cold -> positive side (R17)
    ctx.last_pos, ctx.last_neg = 4, 4  # both < n/3: smaller count, then positive
    assert ctx.select_mode() == L.POS
    ctx.last_pos, ctx.last_neg = 6, 4
    assert ctx.select_mode() == L.NEG


def test_context_negative_side_and_direct():
    rng = np.random.default_rng(21)
    n = 45
    for p, want in ((40, L.NEG), (22, L.DIRECT)):
        lam = np.concatenate([rng.uniform(0.1, 2, p), rng.uniform(-2, -0.1, n - p)])
        Q = haar_q(rng, n)
        A = planted(Q, lam)
        Pstar = (Q * np.maximum(lam, 0)) @ Q.T
        ctx = L.Context(n, seed=4)
        ctx.last_pos, ctx.last_neg = p, n - p
        P, info = ctx.project(A, 1e-10)
        assert info["mode"] == want
        assert np.linalg.norm(P - Pstar) <= 1e-9 * np.linalg.norm(A)


def test_direct_bound_dominates_and_is_tight():
    """R53: the DIRECT path's bound (Theorem 3 with the perp term bounded by the residual of the
    non-positive pairs) dominates the error against LAPACK's projection (an independent routine)
    and stays at the rounding level: eps <= 200 n u ||A||_F."""
    for seed in range(6):
        rng = np.random.default_rng(700 + seed)
        n = int(rng.integers(5, 70))
        M = rng.standard_normal((n, n)) * 10.0 ** rng.uniform(-3, 3)
        A = 0.5 * (M + M.T)
        ctx = L.Context(n, side=L.DIRECT)
        P, info = ctx.project(A, 1e-10)
        w, Vf = np.linalg.eigh(A)
        Pl = (Vf[:, w > 0] * w[w > 0]) @ Vf[:, w > 0].T
        err = np.linalg.norm(P - Pl)
        nA = np.linalg.norm(A)
        assert info["err_bound"] >= err, (seed, err, info["err_bound"])
        assert info["err_bound"] <= 200 * n * L.U * nA


def test_bound_with_perturbed_basis_dominates():
    """R36/R53: the bound's defect terms cover a basis that is neither exactly orthonormal nor
    exactly Rayleigh-Ritz (hard-locked columns frozen while the rest rotate): V = the exact
    positive eigenvectors perturbed by 1e-9 and 1e-6, theta = the exact eigenvalues."""
    rng = np.random.default_rng(41)
    n, p = 50, 6
    lam = np.concatenate([rng.uniform(0.5, 3, p), rng.uniform(-3, -0.5, n - p)])
    Q = haar_q(rng, n)
    A = planted(Q, lam)
    Pstar = (Q * np.maximum(lam, 0)) @ Q.T
    for eta in (1e-9, 1e-6, 1e-4):
        V = Q[:, :p] + eta * rng.standard_normal((n, p))
        th = lam[:p].copy()
        err = np.linalg.norm((V * th) @ V.T - Pstar)
        assert L.error_bound(A, V, th) >= err, (eta, err)


def test_krylov_depth_extension_same_projection_fewer_iterations():
    """R57 (an extension of Alg. 3, off by default): the trial subspace span(X, R, B R, B^2 R, dX)
    reaches the same projection (planted closed form) in fewer iterations on a spectrum with a small
    gap at zero (the C3-R regime), and the Ritz count still interlaces."""
    rng = np.random.default_rng(57)
    n, p = 300, 15
    lam = np.concatenate([10.0 ** rng.uniform(-2, 1, p), -(10.0 ** rng.uniform(-2, 1, n - p))])
    Q = haar_q(rng, n)
    A = planted(Q, lam)
    Pstar = (Q * np.maximum(lam, 0)) @ Q.T
    its = {}
    for d in (1, 3):
        ctx = L.Context(n, seed=3, krylov_depth=d)
        P, info = ctx.project(A, 1e-9)
        assert info["status"] == L.OK and info["npos"] == p
        assert np.linalg.norm(P - Pstar) <= 1e-9 * np.linalg.norm(A)
        assert info["err_bound"] >= np.linalg.norm(P - Pstar)
        its[d] = info["iters"]
    assert its[3] * 1.5 <= its[1], its


def test_krylov_max_active_switches_depth_by_active_width():
    """R63: with krylov_max_active the R57 directions join the basis only on iterations whose active
    set is narrow. A limit at least as wide as the block reproduces R57 on every iteration, a limit
    of 0 columns' worth (1 here, below every active width > 1) stays close to Alg. 3's iteration
    count, an intermediate limit lands in between; every variant reaches the planted projection."""
    rng = np.random.default_rng(63)
    n, p = 300, 15
    lam = np.concatenate([10.0 ** rng.uniform(-2, 1, p), -(10.0 ** rng.uniform(-2, 1, n - p))])
    Q = haar_q(rng, n)
    A = planted(Q, lam)
    Pstar = (Q * np.maximum(lam, 0)) @ Q.T
    its = {}
    for name, kw in (("alg3", dict(krylov_depth=1)), ("r57", dict(krylov_depth=2)),
                     ("wide", dict(krylov_depth=2, krylov_max_active=n)),
                     ("mid", dict(krylov_depth=2, krylov_max_active=22))):
        ctx = L.Context(n, seed=3, **kw)
        P, info = ctx.project(A, 1e-9)
        assert info["status"] == L.OK and info["npos"] == p, name
        assert np.linalg.norm(P - Pstar) <= 1e-9 * np.linalg.norm(A), name
        assert info["err_bound"] >= np.linalg.norm(P - Pstar), name
        its[name] = info["iters"]
    assert its["wide"] == its["r57"], its
    assert its["r57"] <= its["mid"] <= its["alg3"], its
    assert its["mid"] < its["alg3"], its


def test_guard_active_warm_sequence_same_projection():
    """R62 (the GPU default on warm calls): with only the top 2 guards keeping their directions the
    warm projections of a drifting planted sequence still reach the closed form within tolerance, the
    bound dominates, and the positive count is right; cold calls are unaffected (all columns active)."""
    rng = np.random.default_rng(62)
    n, p = 160, 8
    lam = np.concatenate([10.0 ** rng.uniform(-2, 1, p), -(10.0 ** rng.uniform(-2, 1, n - p))])
    Q = haar_q(rng, n)
    ctxs = {ga: L.Context(n, seed=5, guard_active=ga) for ga in (None, 2)}
    for t in range(4):
        K = rng.standard_normal((n, n))
        K = (K - K.T) / (2.0 * np.sqrt(n))
        Qt = np.linalg.qr((np.eye(n) + 1e-3 * K) @ Q)[0] if t else Q
        A = planted(Qt, lam)
        Pstar = (Qt * np.maximum(lam, 0)) @ Qt.T
        for ga, ctx in ctxs.items():
            P, info = ctx.project(A, 1e-9)
            assert info["status"] == L.OK and info["npos"] == p, (t, ga, info)
            err = np.linalg.norm(P - Pstar)
            assert err <= 1e-9 * np.linalg.norm(A), (t, ga, err)
            assert info["err_bound"] >= err, (t, ga)
