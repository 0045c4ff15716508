"""f2 (reading R48): the projected-Lanczos perp term of Theorem 3.

CPU: the oracle's estimate_perp pinned to the SPEC examples, to the exact top
eigenvalue of the deflated operator (numpy eigvalsh on an explicit complement basis: an
independent routine), and to Theorem 3's dominance when the block misses a positive eigenvalue.
GPU: the library's bound with perp_steps > 0 dominates the true error of a projection whose block
missed positive eigenvalues, and the perp term vanishes when every positive pair was found."""
import numpy as np
import pytest
import torch

from oracle.exact import project_exact
from oracle.lobpcg import error_bound, estimate_perp
from workloads.generators import haar_q, planted


def test_perp_spec_examples():
    # V spans the positive eigenspace of diag(1, -1): the deflated operator is NSD -> 0
    mu, r, perp = estimate_perp(np.diag([1.0, -1.0]), np.array([[1.0], [0.0]]), 5)
    assert perp == 0.0 and abs(mu + 1.0) <= 1e-15
    # V = e2 on diag(5, -1): the e1 direction is left -> 5
    mu, r, perp = estimate_perp(np.diag([5.0, -1.0]), np.array([[0.0], [1.0]]), 5)
    assert abs(mu - 5.0) <= 1e-14 and abs(perp - 5.0) <= 1e-13


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_perp_matches_deflated_top_eigenvalue(seed):
    rng = np.random.default_rng(seed)
    n = 40
    Q = haar_q(rng, n)
    lam = np.concatenate([[2.0, 3.0, 4.0, 0.7], -rng.uniform(0.5, 10.0, n - 4)])
    A = planted(Q, lam)
    V = Q[:, [1, 2]]          # the block found 3 and 4, missed 2 and 0.7
    Vc = Q[:, [0, 3] + list(range(4, n))]  # an orthonormal basis of the complement
    top = np.linalg.eigvalsh(Vc.T @ A @ Vc).max()
    mu, r, perp = estimate_perp(A, V, 30, seed=seed)
    assert abs(mu - top) <= r + 1e-12 * abs(top)
    assert mu + r >= top - 1e-12
    assert perp >= np.sqrt(n - 2) * top - 1e-10


def test_perp_makes_the_bound_dominate_a_missed_eigenvalue():
    rng = np.random.default_rng(9)
    n = 30
    Q = haar_q(rng, n)
    lam = np.concatenate([[2.0, 3.0, 4.0], -rng.uniform(1.0, 10.0, n - 3)])
    A = planted(Q, lam)
    V = Q[:, [1, 2]]                       # exact pairs, but the eigenvalue 2 is missed
    theta = np.array([3.0, 4.0])
    err = np.linalg.norm((V * theta) @ V.T - project_exact(A))
    assert abs(err - 2.0) <= 1e-10        # Theorem 3's perp term is the whole error here
    assert error_bound(A, V, theta) < err  # the paper's bound (p^ = 0) does not dominate
    _, _, perp = estimate_perp(A, V, 20)
    assert error_bound(A, V, theta, perp=perp) >= err


def test_perp_invariant_subspace_terminates():
    rng = np.random.default_rng(4)
    n = 12
    Q = haar_q(rng, n)
    lam = np.linspace(-3.0, 2.0, n)
    A = planted(Q, lam)
    V = Q[:, 1:]                           # a one-dimensional complement: one Lanczos step is exact
    mu, r, perp = estimate_perp(A, V, 10)
    assert abs(mu - lam[0]) <= 1e-12 and r <= 1e-12 and perp == 0.0


@pytest.mark.gpu
def test_gpu_perp_bound_dominates(api):
    """A cold block narrower than the positive eigenspace, stopped after one iteration with a
    loose tolerance: positive eigenvalues are missed; with perp_steps the bound still dominates."""
    rng = np.random.default_rng(12)
    n, p = 200, 12
    lam = np.concatenate([rng.uniform(1.0, 5.0, p), -rng.uniform(1.0, 5.0, n - p)])
    A = planted(haar_q(rng, n), lam)
    Pe = project_exact(A)
    for steps in (0, 40):
        ctx = api.Context(n, params=api.default_params(seed=3, m0=4, expand_q=2, max_iter=1, side=1,
                                                        perp_steps=steps))
        Pi, info = ctx.project(torch.from_numpy(A).cuda(), 1e3)
        err = np.linalg.norm(Pi.cpu().numpy() - Pe)
        assert info["npos"] < p, info            # the block missed positives
        if steps == 0:
            assert info["perp_est"] == 0.0
        else:
            assert info["perp_est"] > 0.0
            assert info["err_bound"] >= err, (info["err_bound"], err)
        ctx.close()


@pytest.mark.gpu
def test_gpu_perp_vanishes_when_converged(api):
    rng = np.random.default_rng(13)
    n, p = 150, 10
    lam = np.concatenate([rng.uniform(1.0, 5.0, p), -rng.uniform(1.0, 5.0, n - p)])
    A = planted(haar_q(rng, n), lam)
    ctx = api.Context(n, params=api.default_params(seed=3, perp_steps=40))
    Pi, info = ctx.project(torch.from_numpy(A).cuda(), 1e-10)
    assert info["npos"] == p and info["perp_est"] == 0.0
    assert info["err_bound"] >= np.linalg.norm(Pi.cpu().numpy() - project_exact(A))
    ctx.close()
