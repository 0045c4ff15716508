"""Oracle for f1 / f3 (TEST INFRASTRUCTURE; see oracle/__init__.py): Alg. 1 of PAPER.md:62-83 for
the diagonal SDP  min <Q, X>  s.t.  X_ii = b_i (i with w_i = 1),  X PSD  (MaxCut: Q = -L/4, b = 1,
w = 1), written step by step in the paper's notation with exact projections (O-EXACT,
oracle/exact.py), and the infeasibility certificates of Theorem 1 in the
practical form of PAPER.md:563-587 (reading R49).

Problem in the form of PAPER.md:50-57: minimise q^T x (P = 0) s.t. A x = z, z in C, with
x = vec(X), q = vec(-L/4), A = [D; I] (D picks the diagonal), C = {1}^n x S+.
Line 3: [sigma I, rho A^T; rho A, -rho I] [x~; nu] = [sigma x - q + rho A^T (z - y/rho); 0]
        -> (sigma I + rho A^T A) x~ = sigma x - q + rho A^T (z - y/rho), z~ = A x~
Line 4: x <- alpha x~ + (1 - alpha) x
Line 5: z <- Pi_C(z_hat + y/rho), z_hat = alpha z~ + (1 - alpha) z      (reading R43)
Line 6: y <- y + rho (z_hat - z)
The linear system is solved by its definition (A^T A is formed explicitly as a matrix for small n).
"""
import numpy as np

from .exact import project_exact


def diag_sdp_admm(Q, b=None, w=None, rho=0.1, sigma=1e-6, alpha=1.6, eps=1e-4, max_iter=5000, project=None,
                  keep_last=False, adapt_every=0, adapt_ratio=5.0):
    """Alg. 1 on min <Q, X> s.t. X_ii = b_i (w_i = 1), X PSD. Returns X, objective, iterations, the
    residual history and (keep_last) the last two iterates (x, y) for the certificates."""
    n = Q.shape[0]
    b = np.ones(n) if b is None else np.asarray(b, dtype=np.float64)
    w = np.ones(n) if w is None else np.asarray(w, dtype=np.float64)
    eq = np.flatnonzero(w != 0)
    project = project or project_exact
    N = n * n
    # A = [D_w; I] on vec(X) (column-major vec): D_w picks entries i + i n for the constrained i
    D = np.zeros((eq.size, N))
    D[np.arange(eq.size), eq * (n + 1)] = 1.0
    A = np.vstack([D, np.eye(N)])
    ne = eq.size
    q = Q.reshape(-1, order="F")
    AtA = A.T @ A
    Kinv = np.linalg.inv(sigma * np.eye(N) + rho * AtA)  # line 3's solve is x~ = K^-1 rhs
    rhos = [(0, rho)]
    x = np.zeros(N)
    z = np.concatenate([b[eq], np.zeros(N)])
    y = np.zeros(ne + N)
    hist = []
    prev = None
    k = 0
    for k in range(1, max_iter + 1):
        prev = (x.copy(), y.copy())
        rhs = sigma * x - q + rho * (A.T @ (z - y / rho))
        xt = Kinv @ rhs
        zt = A @ xt
        x = alpha * xt + (1 - alpha) * x
        zh = alpha * zt + (1 - alpha) * z
        v = zh + y / rho
        znew = np.empty_like(z)
        znew[:ne] = b[eq]                                        # projection onto {b}
        Vm = v[ne:].reshape(n, n, order="F")
        znew[ne:] = project(0.5 * (Vm + Vm.T)).reshape(-1, order="F")  # PSD block
        y = y + rho * (zh - znew)
        z = znew
        r_prim = np.abs(A @ x - z).max()
        r_dual = np.abs(q + A.T @ y).max()
        hist.append((r_prim, r_dual))
        if r_prim <= eps and r_dual <= eps:
            break
        # reading R58: residual balancing every adapt_every iterations (COSMO); K changes with rho
        if adapt_every > 0 and k % adapt_every == 0 and r_prim > 0 and r_dual > 0:
            ratio = r_prim / r_dual
            if ratio > adapt_ratio or ratio < 1.0 / adapt_ratio:
                rho = min(1e6, max(1e-6, rho * ratio ** 0.5))
                Kinv = np.linalg.inv(sigma * np.eye(N) + rho * AtA)
                rhos.append((k, rho))
    X = x.reshape(n, n, order="F")
    out = {"X": X, "objective": float(np.sum(Q * X)), "iters": k, "hist": hist, "rhos": rhos}
    if keep_last:
        out.update({"x": x, "y": y, "x_prev": prev[0], "y_prev": prev[1], "A": A, "eq": eq, "b": b, "q": q})
    return out


def maxcut_admm(L, rho=0.1, sigma=1e-6, alpha=1.6, eps=1e-4, max_iter=5000, project=None, adapt_every=0):
    out = diag_sdp_admm(-0.25 * L, rho=rho, sigma=sigma, alpha=alpha, eps=eps, max_iter=max_iter, project=project,
                        adapt_every=adapt_every)
    out["objective"] = -out["objective"]  # max 1/4 <L, X>
    return out


def certificates(run, n):
    """Theorem 1 in the practical form of PAPER.md:563-587, reading R49, from the
    last two iterates of diag_sdp_admm(..., keep_last=True): with y-bar = dy/||dy||, x-bar = dx/||dx||,
      primal: ||A^T y-bar||_inf, dist_{C-polar}(y-bar) = ||Pi_S+(Y-bar)||_F, support b^T y-bar_eq
      dual:   dist_{C-inf}(A x-bar) = sqrt(||diag_w(X-bar)||^2 + ||Pi_S+(-X-bar)||_F^2), q^T x-bar
    (the PSD projections exact, O-EXACT). Returns a dict of the five numbers and the two norms."""
    A, eq, b, q = run["A"], run["eq"], run["b"], run["q"]
    ne = eq.size
    dx = run["x"] - run["x_prev"]
    dy = run["y"] - run["y_prev"]
    out = {"ndx": float(np.linalg.norm(dx)), "ndy": float(np.linalg.norm(dy))}
    if out["ndy"] > 1e-12:
        yb = dy / out["ndy"]
        Yb = yb[ne:].reshape(n, n, order="F")
        out["p_at"] = float(np.abs(A.T @ yb).max())
        out["p_dist"] = float(np.linalg.norm(project_exact(0.5 * (Yb + Yb.T))))
        out["p_supp"] = float(b[eq] @ yb[:ne])
    if out["ndx"] > 1e-12:
        xb = dx / out["ndx"]
        Xb = xb.reshape(n, n, order="F")
        ax = A @ xb
        out["d_dist"] = float(np.sqrt(np.sum(ax[:ne] ** 2) + np.sum(project_exact(-0.5 * (Xb + Xb.T)) ** 2)))
        out["d_qx"] = float(q @ xb)
    return out
