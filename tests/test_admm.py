"""f1: approximate ADMM (Alg. 1) on MaxCut SDPs (BASELINE configs[4]).

CPU: the oracle's ADMM (exact projections) is pinned to closed-form SDP values: one edge (1),
K3 (9/4), K4 (n^2/4 = 4), the 5-cycle (n (1 + cos(pi/n)) / 2), and to feasibility of its answer.
GPU: the library's ADMM (elementwise steps + warm LOBPCG projections with the 10/k^1.01 schedule)
reaches the same values, and with near-exact projections follows the oracle's iterates."""
import numpy as np
import pytest

from oracle.admm import maxcut_admm


def laplacian(n, edges):
    W = np.zeros((n, n))
    for i, j, w in edges:
        W[i, j] = W[j, i] = w
    return np.diag(W.sum(axis=1)) - W


def cycle(n):
    return laplacian(n, [(i, (i + 1) % n, 1.0) for i in range(n)])


def complete(n):
    return laplacian(n, [(i, j, 1.0) for i in range(n) for j in range(i + 1, n)])


CASES = [("edge", laplacian(2, [(0, 1, 1.0)]), 1.0), ("K3", complete(3), 9 / 4), ("K4", complete(4), 4.0),
         ("C5", cycle(5), 5 * (1 + np.cos(np.pi / 5)) / 2)]


@pytest.mark.parametrize("name,L,value", CASES)
def test_oracle_admm_closed_form_values(name, L, value):
    res = maxcut_admm(L, eps=1e-7, max_iter=20000)
    X = res["X"]
    assert abs(res["objective"] - value) <= 1e-4 * max(1.0, value), (name, res["objective"], value, res["iters"])
    assert np.abs(np.diag(X) - 1).max() <= 1e-5
    assert np.linalg.eigvalsh(0.5 * (X + X.T)).min() >= -1e-5


def test_oracle_admm_residuals_decrease():
    rng = np.random.default_rng(3)
    n = 12
    edges = [(i, j, rng.choice([-1.0, 1.0])) for i in range(n) for j in range(i + 1, n) if rng.uniform() < 0.4]
    res = maxcut_admm(laplacian(n, edges), eps=1e-6, max_iter=5000)
    h = np.array(res["hist"])
    assert h[-1].max() <= 1e-6
    assert h[len(h) // 2:].max() <= h[:len(h) // 4].max()


def test_oracle_adaptive_rho_same_answer():
    """R58: residual balancing every 40 iterations reaches the same SDP values as fixed rho = 0.1 (the
    closed-form cases, and a random +-1 graph at eps 1e-6)."""
    for name, L, value in CASES:
        res = maxcut_admm(L, eps=1e-7, max_iter=20000, adapt_every=40)
        assert abs(res["objective"] - value) <= 1e-4 * max(1.0, value), (name, res["objective"], value)
    rng = np.random.default_rng(3)
    n = 12
    edges = [(i, j, rng.choice([-1.0, 1.0])) for i in range(n) for j in range(i + 1, n) if rng.uniform() < 0.4]
    fixed = maxcut_admm(laplacian(n, edges), eps=1e-6, max_iter=20000)
    adap = maxcut_admm(laplacian(n, edges), eps=1e-6, max_iter=20000, adapt_every=40)
    assert max(adap["hist"][-1]) <= 1e-6
    assert abs(adap["objective"] - fixed["objective"]) <= 1e-4 * abs(fixed["objective"])


@pytest.mark.gpu
@pytest.mark.parametrize("name,L,value", CASES[1:])
def test_gpu_admm_closed_form_values(api, name, L, value):
    from paper_1912_02767_b200.admm import MaxCutADMM
    solver = MaxCutADMM(L)
    out = solver.solve(eps=1e-7, max_iter=20000)
    assert abs(out["objective"] - value) <= 1e-4 * max(1.0, value), (name, out)
    solver.close()


@pytest.mark.gpu
def test_gpu_admm_follows_oracle_iterates(api):
    """Near-exact projections (tol 1e-12): the GPU iterates track the oracle's exact-projection
    ADMM (ADMM's operator is averaged, so the projection errors do not grow)."""
    from paper_1912_02767_b200.admm import MaxCutADMM
    from workloads.generators import maxcut_graph
    L = maxcut_graph(n=30, p_edge=0.3, seed=7)
    ref = maxcut_admm(L, eps=0.0, max_iter=150)
    solver = MaxCutADMM(L, tol_override=1e-12)
    for _ in range(150):
        solver.step()
    X = solver.X.cpu().numpy()
    assert np.linalg.norm(X - ref["X"]) <= 1e-7 * np.linalg.norm(ref["X"])
    solver.close()


@pytest.mark.gpu
def test_gpu_admm_adaptive_follows_oracle_iterates(api):
    """R58 on both sides (residual balancing every 40 iterations): near-exact projections track the
    oracle through the rho changes."""
    from paper_1912_02767_b200.admm import MaxCutADMM
    from workloads.generators import maxcut_graph
    L = maxcut_graph(n=30, p_edge=0.3, seed=7)
    ref = maxcut_admm(L, eps=0.0, max_iter=200, adapt_every=40)
    solver = MaxCutADMM(L, tol_override=1e-12, adapt_every=40)
    for _ in range(200):
        solver.step()
    assert [r for _, r in solver.rho_history] == pytest.approx([r for _, r in ref["rhos"]], rel=1e-12)
    X = solver.X.cpu().numpy()
    assert np.linalg.norm(X - ref["X"]) <= 1e-7 * np.linalg.norm(ref["X"])
    solver.close()


@pytest.mark.gpu
def test_gpu_admm_schedule_converges_c5_small(api):
    """configs[4] recipe at reduced size (n = 200, p = 0.05): with the projection tolerance tied to the
    ADMM residual (R59: min(10/k^1.01, 0.01 min(r_prim, r_dual)); the paper's summable schedule stays
    the upper bound) both residuals reach 1e-4 (R33) in a few hundred iterations; with the paper's
    schedule alone the dual residual reaches 1e-4 and the primal one ~3e-4 within 3000 iterations
    (measured 5222 iterations to 1e-4; 3.03e-4 at 3000 with R62's warm guard directions). The answer is nearly PSD and the LOBPCG calls stay warm."""
    from paper_1912_02767_b200.admm import MaxCutADMM
    from workloads.generators import maxcut_graph
    L = maxcut_graph(n=200, p_edge=0.05, seed=501)
    solver = MaxCutADMM(L, tol_ratio=0.01)
    out = solver.solve(eps=1e-4, max_iter=3000)
    assert out["r_prim"] <= 1e-4 and out["r_dual"] <= 1e-4 and out["iters"] < 1000, out
    X = solver.X.cpu().numpy()
    assert np.linalg.eigvalsh(0.5 * (X + X.T)).min() >= -1e-3
    assert sum(i["cold"] for i in solver.infos) <= 2       # warm starts across ADMM iterations
    solver.close()
    paper = MaxCutADMM(L)
    out2 = paper.solve(eps=1e-4, max_iter=3000)
    assert out2["r_dual"] <= 1e-4 and out2["r_prim"] <= 4e-4, out2
    assert abs(out2["objective"] - out["objective"]) <= 1e-3 * abs(out["objective"])
    paper.close()


# ---------------------------------------------------------------- f3: infeasibility certificates
def _toys(n=6, seed=0):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n))
    Q = 0.5 * (M + M.T)
    b = np.ones(n)
    b[0] = -1.0  # X_00 = -1 with X PSD: primal infeasible
    return Q, b, np.zeros(n)  # w = 0 (no equality rows) with an indefinite Q: dual infeasible


def test_oracle_primal_infeasibility_certificate():
    """Theorem 1 (i): dy -> a certificate with A^T y = 0, S_C(y) < 0, met in the
    practical form of PAPER.md:582-587 at 1e-4 (R49); the direction is the diagonal row of the
    offending constraint (b^T y-bar -> -1/sqrt(2): y_eq = -e_0 / sqrt 2, Y = e_0 e_0^T / sqrt 2 ... up
    to the rest of the cone)."""
    from oracle.admm import certificates, diag_sdp_admm
    Q, b, _ = _toys()
    run = diag_sdp_admm(Q, b=b, eps=0.0, max_iter=800, keep_last=True)
    c = certificates(run, Q.shape[0])
    assert c["ndy"] > 1e-3                                  # dy does not vanish
    assert c["p_at"] < 1e-4 and c["p_dist"] < 1e-4 and c["p_supp"] < -1e-4
    assert abs(c["p_supp"] + 1 / np.sqrt(2)) < 1e-3
    assert not (c["d_dist"] < 1e-4 and c["d_qx"] < -1e-4)  # not dual infeasible


def test_oracle_dual_infeasibility_certificate():
    """Theorem 1 (ii): dx -> a direction with A dx in C^inf (PSD, no equality rows) and q^T dx < 0."""
    from oracle.admm import certificates, diag_sdp_admm
    Q, _, w = _toys()
    run = diag_sdp_admm(Q, w=w, eps=0.0, max_iter=400, keep_last=True)
    c = certificates(run, Q.shape[0])
    assert c["ndx"] > 1.0
    assert c["d_dist"] < 1e-4 and c["d_qx"] < -1e-4
    # the unbounded direction is the normalised steepest descent ray in the cone, Pi_S+(-Q) / ||.||:
    # q^T x-bar -> -||Pi_S+(-Q)||_F = -(sum of the squared negative eigenvalues of Q)^(1/2)
    lam = np.linalg.eigvalsh(Q)
    assert abs(c["d_qx"] + np.sqrt(np.sum(lam[lam < 0] ** 2))) < 1e-3


def test_oracle_feasible_problem_never_certifies():
    from oracle.admm import certificates, diag_sdp_admm
    L = cycle(6)
    for it in (40, 80, 120, 400):
        c = certificates(diag_sdp_admm(-0.25 * L, eps=0.0, max_iter=it, keep_last=True), 6)
        p = "p_at" in c and c["p_at"] < 1e-4 and c["p_dist"] < 1e-4 and c["p_supp"] < -1e-4
        d = "d_dist" in c and c["d_dist"] < 1e-4 and c["d_qx"] < -1e-4
        assert not (p or d), (it, c)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["primal", "dual", "feasible"])
def test_gpu_admm_infeasibility_detection(api, kind):
    """f3: the library's ADMM with approximate (LOBPCG) projections stops on Theorem 1's
    certificate for the infeasible toys and never for a feasible MaxCut."""
    from paper_1912_02767_b200.admm import DiagSDPADMM
    Q, b, w = _toys()
    if kind == "primal":
        solver = DiagSDPADMM(Q, b=b)
    elif kind == "dual":
        solver = DiagSDPADMM(Q, w=w)
    else:
        solver = DiagSDPADMM(-0.25 * cycle(6))
    out = solver.solve(eps=1e-7, max_iter=4000, check_every=40)
    if kind == "primal":
        assert out["status"] == "primal_infeasible", out
        assert abs(out["certificates"]["p_supp"] + 1 / np.sqrt(2)) < 1e-2
    elif kind == "dual":
        assert out["status"] == "dual_infeasible", out
        lam = np.linalg.eigvalsh(Q)
        assert abs(out["certificates"]["d_qx"] + np.sqrt(np.sum(lam[lam < 0] ** 2))) < 1e-2
    else:
        assert out["status"] == "solved", out
    solver.close()
