"""Oracle for f1 (TEST INFRASTRUCTURE; see oracle/__init__.py): Alg. 1 of PAPER.md:62-83 for the
MaxCut SDP  max 1/4 <L, X>  s.t.  diag(X) = 1,  X PSD,  written step by step in the paper's
notation with exact projections (O-EXACT, oracle/exact.py).

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


def maxcut_admm(L, rho=0.1, sigma=1e-6, alpha=1.6, eps=1e-4, max_iter=5000, project=None):
    n = L.shape[0]
    project = project or project_exact
    N = n * n
    # A = [D; I] on vec(X) (column-major vec): D picks entries i + i n
    D = np.zeros((n, N))
    D[np.arange(n), np.arange(n) * (n + 1)] = 1.0
    A = np.vstack([D, np.eye(N)])
    q = (-0.25 * L).reshape(-1, order="F")
    K = sigma * np.eye(N) + rho * (A.T @ A)
    Kinv = np.linalg.inv(K)  # K is fixed across iterations; line 3's solve is x~ = K^-1 rhs
    x = np.zeros(N)
    z = np.concatenate([np.ones(n), np.zeros(N)])
    y = np.zeros(n + N)
    hist = []
    k = 0
    for k in range(1, max_iter + 1):
        rhs = sigma * x - q + rho * (A.T @ (z - y / rho))
        xt = Kinv @ rhs
        zt = A @ xt
        x = alpha * xt + (1 - alpha) * x
        zh = alpha * zt + (1 - alpha) * z
        v = zh + y / rho
        znew = np.empty_like(z)
        znew[:n] = 1.0                                           # projection onto {1}^n
        Vm = v[n:].reshape(n, n, order="F")
        znew[n:] = project(0.5 * (Vm + Vm.T)).reshape(-1, order="F")  # PSD block
        y = y + rho * (zh - znew)
        z = znew
        r_prim = np.abs(A @ x - z).max()
        r_dual = np.abs(q + A.T @ y).max()
        hist.append((r_prim, r_dual))
        if r_prim <= eps and r_dual <= eps:
            break
    X = x.reshape(n, n, order="F")
    return {"X": X, "objective": 0.25 * float(np.sum(L * X)), "iters": k, "hist": hist}
