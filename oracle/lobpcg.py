"""O-LOBPCG: the paper's approximate projection, step by step (TEST INFRASTRUCTURE;
see oracle/__init__.py).

Follows PAPER.md in its order and notation:
  rayleigh_ritz   Alg. 2: orthonormalize S, eig of S^T A S, Ritz pairs.
  cholesky_qr     PAPER.md:395-397 (Cholesky QR, Householder QR fallback [Stewart1998 p.251]).
  lobpcg_pos      Alg. 3 for the positive eigenpairs of B, with the
                  residual-form basis (footnote PAPER.md:377), random expansion (PAPER.md:379-397,
                  line 8), stopping rule (PAPER.md:493 / :507) and locking (BLOPEX active mask,
                  PAPER.md:502; optional hard locking, R35).
  error_bound     Theorem 3 with the perp term ignored.
  perp_bound      f2 (R48): k-step Lanczos on the deflated operator (I - V V^T) B (I - V V^T)
                  ("projected Lanczos") turned into a randomized upper bound on
                  lambda_max (Kuczynski-Wozniakowski), p^ = sqrt(n - p) max(ub, 0).
  direct_bound    the bound of a full eigendecomposition (DIRECT path, R53).
  Context.project the side rule, negation and
                  Pi = V L V^T or A - V L V^T (R4).

Readings of silent / ambiguous passages are numbered R1..R36 in DESIGN.md §3 and cited
inline. Library primitives used as single steps: numpy matmul, numpy Householder QR
(LAPACK geqrf, the paper's own fallback), triangular solve; every eigendecomposition is the
cyclic Jacobi of oracle/jacobi.c.
"""
import math

import numpy as np

from ._clib import cholesky as _chol
from ._clib import jacobi_eig
from .philox import gaussian_block

U = 2.0 ** -53

NOT_CONVERGED = 1
OK = 0


class RankDeficient(Exception):
    """Cholesky QR signalled a (numerically) rank-deficient Gram matrix."""


# --------------------------------------------------------------------------- basics
def eig_desc(H):
    """Symmetric eigendecomposition by Jacobi, ordered descending (Alg. 3 keeps 'the m
    largest'; ties broken by index, R21)."""
    H = 0.5 * (H + H.T)
    w, V, _ = jacobi_eig(H)
    order = np.argsort(-w, kind="stable")
    return w[order], V[:, order]


def cholesky_qr(S, fail_rel=1e-12):
    """Q = S L^-T with L = chol(S^T S). A pivot <= 1e-12 * max diag(G)
    raises RankDeficient (reading R20)."""
    G = S.T @ S
    G = 0.5 * (G + G.T)
    if G.shape[0] == 0:
        return S.copy(), np.zeros((0, 0))
    L, rc = _chol(G, pivot_floor=fail_rel * max(float(np.max(np.diag(G))), 0.0))
    if L is None:
        raise RankDeficient(rc)
    Q = np.linalg.solve(L, S.T).T  # S L^-T
    return Q, L


def householder_qr(S, drop_rel=1e-10):
    """The paper's fallback orthonormalization ('Householder QR'); columns
    whose |R_jj| <= drop_rel * max |R_ii| are dropped (R20)."""
    Q, R = np.linalg.qr(S, mode="reduced")
    d = np.abs(np.diag(R))
    if d.size == 0:
        return Q
    keep = d > drop_rel * d.max()
    return Q[:, keep]


def orthonormalize(S):
    try:
        Q, _ = cholesky_qr(S)
        # CholQR2 when the first pass lost orthogonality (R20)
        if np.linalg.norm(Q.T @ Q - np.eye(Q.shape[1])) > 1e-12:
            Q, _ = cholesky_qr(Q)
        return Q
    except RankDeficient:
        return householder_qr(S)


def rayleigh_ritz(A, S):
    """Alg. 2: Ritz vectors S W~ and Ritz values L~ (ascending) of A on
    span(S)."""
    Q = orthonormalize(S)
    H = Q.T @ (A @ Q)
    w, W, _ = jacobi_eig(0.5 * (H + H.T))
    return Q @ W, w


def residual_norms(A, V, theta):
    """r_i = ||A v_i - theta_i v_i||_2, columns of R = A V~ - V~ L~ (R13)."""
    return np.linalg.norm(A @ V - V * theta, axis=0)


def _unit_cols(M):
    nr = np.linalg.norm(M, axis=0)
    nr[nr == 0] = 1.0
    return M / nr, nr


# --------------------------------------------------------------------------- LOBPCG
class LobpcgResult:
    pass


def lobpcg_pos(B, X0, tol, max_iter=500, guard=1, q=None, locking="hard", seed=0, ctx=0,
               call=0, cold=False, guard_tol=None, m_max=None, lock_factor=1.0, krylov_depth=1, guard_active=None,
               krylov_max_active=0):
    """Alg. 3: positive eigenpairs of the symmetric matrix B.

    X0      n x m start block (warm: previous Ritz block, R27; cold: Philox, R28).
    tol     absolute per-pair residual 2-norm threshold (R12, R13).
    guard   g >= 1 non-positive guard columns kept in the block (R8, R12).
    q       expansion quantum, default max(ceil(0.05 n), 1) (R9).
    locking 'soft' = BLOPEX active mask (X stays whole in the RR basis);
            'hard' = converged positive columns leave the RR basis (R35).
    m_max   block-width capacity; an expansion beyond it stops the iteration with
            abort_direct set (the caller switches to the full eigendecomposition, R18).
    Returns a LobpcgResult with X (n x m), theta (m), r (m), status, iters, counters.
    """
    n = B.shape[0]
    m_max = n if m_max is None else m_max
    q = q if q else max(int(math.ceil(0.05 * n)), 1)
    # guard certification theta_g + r_g <= guard_tol and r_g <= max(guard_tol, |theta_g|/2) (R52, R60)
    guard_tol = tol if guard_tol is None else guard_tol
    res = LobpcgResult()
    res.expansions = 0
    res.a_passes = 0
    res.a_cols = 0
    res.trace = []  # per iteration: (basis width s, active |J|, locked count, positives)

    def mul(Z):
        res.a_passes += 1
        res.a_cols += Z.shape[1]
        return B @ Z

    # Alg. 3 line 2: (L0, X0) <- Rayleigh-Ritz on span(X0)
    X = orthonormalize(X0)
    BX = mul(X)
    theta, C = eig_desc(X.T @ BX)
    X = X @ C
    BX = BX @ C
    m = X.shape[1]
    # line 3: Delta X^0 empty. P/BP hold one direction per block column (R5, BLOPEX form)
    P = np.zeros((n, m))
    BP = np.zeros((n, m))
    has_p = np.zeros(m, dtype=bool)
    locked = np.zeros(m, dtype=bool)
    r = np.full(m, np.inf)
    E = None  # pending expansion columns (orthonormal, ⟂ X)
    status = NOT_CONVERGED
    k = 0
    abort_direct = False
    while True:
        # line 5: R^k = A X^k - X^k L^k (residual form, footnote PAPER.md:377)
        R = BX - X * theta
        ul = ~locked
        r[ul] = np.linalg.norm(R[:, ul], axis=0)
        # stopping rule (R12): every positive Ritz pair r_i <= tol AND guard
        pos = theta > 0
        conv_pos = bool(np.all(r[pos] <= tol))
        npos = int(np.sum(pos))
        if m >= n:
            guard_ok = True
        elif npos >= m:
            guard_ok = False
        else:
            g = int(np.argmax(np.where(pos, -np.inf, theta)))
            # R52 relaxed form, R60: the guard itself must be within max(tol, |theta_g|/2) of convergence
            guard_ok = bool(theta[g] + r[g] <= guard_tol and r[g] <= max(guard_tol, 0.5 * abs(theta[g])))
        converged = conv_pos and guard_ok and E is None and not (cold and k == 0)
        if converged:
            status = OK
            break
        if k >= max_iter:
            break
        # locking (R35): hard mode locks converged positive pairs
        if locking == "hard":
            locked |= pos & (r <= lock_factor * tol)  # R55
        Uidx = np.flatnonzero(~locked)
        Lidx = np.flatnonzero(locked)
        # active set J (BLOPEX active mask): unlocked columns with r_i > tol
        J = Uidx[r[Uidx] > tol]
        if guard_active is not None and guard_active >= 0 and not cold:
            # R62 (option; the GPU default on warm calls): only the guard_active largest non-positive
            # Ritz values keep their directions (theta is sorted descending)
            npu = Uidx[theta[Uidx] <= 0]
            keep = set(npu[np.argsort(-theta[npu], kind="stable")][:guard_active].tolist())
            J = np.array([j for j in J if theta[j] > 0 or j in keep], dtype=J.dtype)
        if locking == "soft":
            Xs, BXs, thetas = X, BX, theta
            Sidx = np.arange(m)
        else:
            Xs, BXs, thetas = X[:, Uidx], BX[:, Uidx], theta[Uidx]
            Sidx = Uidx
        W = R[:, J]
        if E is not None:
            W = np.hstack([W, E])
        XL = X[:, Lidx]
        if locking == "hard" and XL.shape[1]:
            W = W - XL @ (XL.T @ W)
        W, _ = _unit_cols(W)
        BW = mul(W) if W.shape[1] else np.zeros((n, 0))
        PJ = J[has_p[J]]
        Pm, BPm = P[:, PJ], BP[:, PJ]
        if locking == "hard" and XL.shape[1] and Pm.shape[1]:
            cP = XL.T @ Pm
            Pm = Pm - XL @ cP
            BPm = BPm - BX[:, Lidx] @ cP
        Pm, pn = _unit_cols(Pm)
        BPm = BPm / pn
        # R57 (an extension, not Alg. 3): block-Krylov directions K_k = B K_{k-1} (K_1 = the normalised
        # R_J), each projected against X_L, X_U and R_J and normalised, appended after P
        a = len(J)
        Kb, BKb = [], []
        prev = BW[:, :a]
        # R63: only on iterations whose active set has at most krylov_max_active columns (0: always)
        depth = 1 if (krylov_max_active > 0 and a > krylov_max_active) else krylov_depth
        for _ in range(1, depth if a else 1):
            K = prev.copy()
            if locking == "hard" and XL.shape[1]:
                K = K - XL @ (XL.T @ K)
            K = K - Xs @ (Xs.T @ K)
            K = K - W[:, :a] @ (W[:, :a].T @ K)
            K, _ = _unit_cols(K)
            BK = mul(K)
            Kb.append(K)
            BKb.append(BK)
            prev = BK
        if Kb:
            Pm = np.hstack([Pm] + Kb)
            BPm = np.hstack([BPm] + BKb)
        mU = Xs.shape[1] + (E.shape[1] if E is not None else 0)
        E = None
        # line 6: Rayleigh-Ritz on span(X, R, P) (R6: P empty at k = 0) via Cholesky QR
        rr = None
        for use_p in (True, False):
            S = np.hstack([Xs, W, Pm]) if use_p else np.hstack([Xs, W])
            BS = np.hstack([BXs, BW, BPm]) if use_p else np.hstack([BXs, BW])
            G = S.T @ S
            H = S.T @ BS
            kx = Xs.shape[1]
            # known blocks inserted exactly (X^T X = I, X^T B X = Theta)
            G[:kx, :kx] = np.eye(kx)
            H[:kx, :kx] = np.diag(thetas)
            G = 0.5 * (G + G.T)
            H = 0.5 * (H + H.T)
            Lc, rc = _chol(G, pivot_floor=1e-12 * max(float(np.max(np.diag(G))), 0.0))
            if Lc is None:
                continue
            Li = np.linalg.solve(Lc, np.eye(G.shape[0]))
            Hh = Li @ H @ Li.T
            th, Ch = eig_desc(Hh)
            Cp = Li.T @ Ch  # C' = L^-T C
            rr = (S, BS, th, Cp, kx)
            res.trace.append((S.shape[1], len(J), int(np.sum(locked)), npos))
            break
        if rr is None:
            # Householder QR fallback
            S = np.hstack([Xs, W, Pm])
            Q = householder_qr(S)
            BQ = mul(Q)
            th, Ch = eig_desc(Q.T @ BQ)
            mU = min(mU, Q.shape[1])
            Xn = Q @ Ch[:, :mU]
            BXn = BQ @ Ch[:, :mU]
            Pn = Xn - Xs @ (Xs.T @ Xn)
            BPn = BXn - BXs @ (Xs.T @ Xn)
            rr_fb = True
        else:
            S, BS, th, Cp, kx = rr
            mU = min(mU, S.shape[1])
            C1 = Cp[:, :mU]
            Xn = S @ C1
            BXn = BS @ C1
            # P = the [R P]-component of the update (R5; BLOPEX form of Delta X)
            Pn = S[:, kx:] @ C1[kx:, :]
            BPn = BS[:, kx:] @ C1[kx:, :]
            rr_fb = False
        # positive Ritz count among all RR values (+ locked ones) -> expansion test (R8)
        p_rr = int(np.sum(th > 0)) + int(np.sum(locked)) if locking == "hard" else int(np.sum(th > 0))
        th_n = th[:mU]
        # assemble the new block: locked columns stay, unlocked replaced by the RR output
        if locking == "hard":
            Xnew = np.hstack([X[:, Lidx], Xn])
            BXnew = np.hstack([BX[:, Lidx], BXn])
            thnew = np.concatenate([theta[Lidx], th_n])
            rnew = np.concatenate([r[Lidx], np.full(mU, np.inf)])
            lnew = np.concatenate([np.ones(len(Lidx), bool), np.zeros(mU, bool)])
            Pnew = np.hstack([np.zeros((n, len(Lidx))), Pn])
            BPnew = np.hstack([np.zeros((n, len(Lidx))), BPn])
            hpnew = np.concatenate([np.zeros(len(Lidx), bool), np.ones(mU, bool)])
        else:
            Xnew, BXnew, thnew = Xn, BXn, th_n
            rnew = np.full(mU, np.inf)
            lnew = np.zeros(mU, bool)
            Pnew, BPnew = Pn, BPn
            hpnew = np.ones(mU, bool)
        if rr_fb:
            hpnew[:] = False
        X, BX, theta, r, locked, P, BP, has_p = Xnew, BXnew, thnew, rnew, lnew, Pnew, BPnew, hpnew
        m = X.shape[1]
        k += 1
        # line 8: expand with random vectors when the positive count leaves < g guards (R8-R11)
        if p_rr >= m - guard + 1 and m < n:
            qq = min(q, n - m)
            if m + qq > m_max:
                abort_direct = True
                break
            Ez = gaussian_block(n, qq, seed, stream=call, ctx=ctx, tag=k)
            for _ in range(2):
                Ez = Ez - X @ (X.T @ Ez)
            E = orthonormalize(Ez)
            res.expansions += 1
            m_target = m + E.shape[1]
            res.m_target = m_target
    res.status = status
    res.iters = k
    res.abort_direct = abort_direct
    # order the block descending
    order = np.argsort(-theta, kind="stable")
    res.X = X[:, order]
    res.BX = BX[:, order]
    res.theta = theta[order]
    res.r = r[order]
    res.m = X.shape[1]
    return res


def error_bound(B, V, theta, perp=0.0, delta_fp=None):
    """Theorem 3 for the positive Ritz pairs (V, theta>0), certified from an
    explicit B V (reading R16), with the perp term p^ (0 = the paper's choice; R14):

      eps = (1 + e) sqrt(2 ||R+||_F^2 + p^2) + (1 + sqrt 2) d + 7 e theta_max + delta_fp

    R+ = B V+ - V+ Theta+, d = ||V+^T B V+ - Theta+||_F (zero for an exact Rayleigh-Ritz output;
    the hard-locking term, R36), e = ||V+^T V+ - I||_F (R53) and delta_fp = 4 n u ||B||_F (R15).
    Derivation (R36/R53): Theorem 3 holds for (V, H = V^T B V) whatever the basis of
    span(V); ||V Theta V^T - V H V^T|| <= d and ||B V - V H|| <= ||R+|| + d give the d terms; the
    polar factor of a nearly orthonormal V moves V Theta V^T by <= e theta_max (2 + e)."""
    n = B.shape[0]
    pos = theta > 0
    Vp = V[:, pos]
    tp = theta[pos]
    BVp = B @ Vp
    R = BVp - Vp * tp
    d = float(np.linalg.norm(Vp.T @ BVp - np.diag(tp)))
    e = float(np.linalg.norm(Vp.T @ Vp - np.eye(Vp.shape[1])))
    thmax = float(np.max(tp)) if tp.size else 0.0
    if delta_fp is None:
        delta_fp = 4 * n * U * np.linalg.norm(B)
    return ((1 + e) * math.sqrt(2 * float(np.sum(R * R)) + perp ** 2) + (1 + math.sqrt(2)) * d
            + 7 * e * thmax + delta_fp)


def direct_bound(A, V, w):
    """Bound for a full eigendecomposition (the DIRECT path, reading R53): Theorem 3 with V~ = the
    eigenvectors of the positive eigenvalues; its perp term is at most (1 + e) ||A V- - V- w-||_F,
    because Pi(V-^T A V-) is the distance of V-^T A V- to the NSD cone, at most its distance
    ||V-^T A V- - diag(w-)||_F to the NSD matrix diag(w-) (w- <= 0), and that is <= ||V-|| ||R-||_F.
    e is the orthonormality defect of the whole basis ||V^T V - I||_F."""
    pos = w > 0
    Rn = A @ V[:, ~pos] - V[:, ~pos] * w[~pos]
    e = float(np.linalg.norm(V.T @ V - np.eye(V.shape[1])))
    perp = (1 + e) * float(np.linalg.norm(Rn))
    return error_bound(A, V, w, perp=perp)


def perp_bound(B, V, steps, seed=0, stream=0, ctx=0, tag=0xC0000000, delta=1e-6, start=None):
    """f2, reading R48 (revised): an upper bound on the perp term of Theorem 3 (
    ignored by the paper, :508, which names "a projected Lanczos algorithm" for it),
    ||Pi(V_perp^T B V_perp)||_F <= sqrt(n - p) max(lambda_max(D), 0), D = B on span(V)^perp.

    `steps` Lanczos steps on D = (I - V V^T) B (I - V V^T) from a Philox start (stream, ctx, tag as
    the library; `start` overrides it, for tests), full reorthogonalisation (two classical
    Gram-Schmidt passes against V and the Lanczos basis); mu = the largest eigenvalue of T_k
    (cyclic Jacobi). Kuczynski & Wozniakowski (1992): for a PSD M of order N and a start uniform on
    the sphere, P{xi_k < (1 - eps) lambda_1(M)} <= 1.648 sqrt(N) exp(-sqrt(eps) (2k - 1)). With
    M = D - c I, c = -||B||_F <= lambda_min(D), with probability >= 1 - delta:
        lambda_max(D) <= c + (mu - c) / (1 - eps),  sqrt(eps) = ln(1.648 sqrt(N) / delta) / (2k - 1);
    eps >= 1 gives the trivial lambda_max(D) <= ||B||_F. A breakdown (invariant Krylov space) or
    k = N makes mu = lambda_max(D) itself (a random start meets every eigenspace). The guarantee is
    over the draw of the start: a matrix built against a known start can defeat it.
    Returns (mu, ub, p^); an empty complement or steps = 0 gives (0, 0, 0)."""
    n = B.shape[0]
    p = V.shape[1]
    N = n - p
    k = min(int(steps), N)
    if k <= 0:
        return 0.0, 0.0, 0.0

    def deflate(w, Q):
        for _ in range(2):
            if p:
                w = w - V @ (V.T @ w)
            if Q.shape[1]:
                w = w - Q @ (Q.T @ w)
        return w

    q = gaussian_block(n, 1, seed, stream, ctx=ctx, tag=tag)[:, 0] if start is None else np.array(start, float)
    q = deflate(q, np.zeros((n, 0)))
    q = q / np.linalg.norm(q)
    Q = q[:, None]
    alpha, beta = [], []
    anorm = float(np.linalg.norm(B))
    breakdown = False
    for j in range(k):
        w = B @ Q[:, j]
        if p:
            w = w - V @ (V.T @ w)
        alpha.append(float(Q[:, j] @ w))
        w = deflate(w, Q)
        b = float(np.linalg.norm(w))
        beta.append(b)
        if b <= 1e-14 * max(anorm, 1e-300):
            breakdown = True
            break
        if j == k - 1:
            break
        Q = np.column_stack([Q, w / b])
    kk = len(alpha)
    T = np.diag(alpha)
    for i in range(kk - 1):
        T[i, i + 1] = T[i + 1, i] = beta[i]
    w_, _, _ = jacobi_eig(T)
    mu = float(np.max(w_))
    if breakdown or kk >= N:
        ub = mu + 4 * kk * U * anorm
    else:
        se = math.log(1.648 * math.sqrt(N) / delta) / (2 * kk - 1)
        eps = se * se
        c = -anorm
        ub = anorm if eps >= 1 else min(anorm, c + (mu - c) / (1 - eps))
    return mu, ub, math.sqrt(N) * max(ub, 0.0)


# --------------------------------------------------------------------------- context
POS, NEG, DIRECT = 1, -1, 2


class Context:
    """Projection context across ADMM iterations: the side rule state and
    the warm block. One per cone block."""

    def __init__(self, n, tol_default=1e-8, max_iter=500, guard=1, q=None, m0=None,
                 locking="hard", seed=0, ctx_id=0, side=0, keep_extra=None, krylov_depth=1, guard_active=None,
                 krylov_max_active=0):
        self.n = n
        self.max_iter = max_iter
        self.guard = guard
        self.q = q
        self.m0 = m0 if m0 else max(int(math.ceil(0.1 * n)), 1)  # R28
        self.locking = locking
        self.seed = seed
        self.ctx_id = ctx_id
        self.side_param = side
        self.keep_extra = keep_extra
        self.krylov_depth = krylov_depth
        self.guard_active = guard_active
        self.krylov_max_active = krylov_max_active
        # capacity ceil(n/3)+1: a wider block is the exact-eig regime (R18)
        self.m_max = min(n, (n + 2) // 3 + 1)
        self.reset()

    def reset(self):
        self.last_pos = None
        self.last_neg = None
        self.X = None
        self.block_side = 0
        self.calls = 0

    def select_mode(self):
        """PAPER.md:505 ('less than a third'), strict < n/3 (R17); ties -> smaller count,
        then positive; cold -> side hint else positive (R17)."""
        if self.side_param in (POS, NEG, DIRECT):
            return self.side_param
        n = self.n
        if self.last_pos is None:
            return POS
        pos_ok = self.last_pos < n / 3
        neg_ok = self.last_neg < n / 3
        if pos_ok and neg_ok:
            return POS if self.last_pos <= self.last_neg else NEG
        if pos_ok:
            return POS
        if neg_ok:
            return NEG
        return DIRECT

    def _keep(self, theta, m):
        p = int(np.sum(theta > 0))
        # R37 revised (R56): a guard band of at least 16 columns beyond the positives
        extra = self.keep_extra if self.keep_extra is not None else max(self.guard, int(math.ceil(0.1 * p)), 16)
        return min(m, p + extra)

    def project(self, A, tol):
        """One projection call: returns (Pi, info dict)."""
        A = np.asarray(A, dtype=np.float64)
        n = self.n
        mode = self.select_mode()
        call = self.calls
        self.calls += 1
        info = dict(mode=mode, call=call)
        if mode != DIRECT and 3 * (self.X.shape[1] if (self.X is not None and self.block_side == mode) else self.m0) >= n:
            mode = DIRECT  # R18: 3m >= n
            info["mode"] = mode
        if mode != DIRECT:
            s = 1.0 if mode == POS else -1.0
            B = s * A
            cold = not (self.X is not None and self.block_side == mode)
            X0 = gaussian_block(n, self.m0, self.seed, stream=call, ctx=self.ctx_id, tag=0) if cold else self.X
            res = lobpcg_pos(B, X0, tol, max_iter=self.max_iter, guard=self.guard, q=self.q,
                             locking=self.locking, seed=self.seed, ctx=self.ctx_id, call=call,
                             cold=cold, m_max=self.m_max, krylov_depth=self.krylov_depth,
                             guard_active=self.guard_active, krylov_max_active=self.krylov_max_active)
            if res.abort_direct:
                mode = DIRECT
                info["mode"] = mode
                info["aborted_to_direct"] = True
            else:
                pos = res.theta > 0
                V = res.X[:, pos]
                th = res.theta[pos]
                lowrank = (V * th) @ V.T
                Pi = lowrank if s > 0 else A + lowrank  # PAPER.md:317 / :319 (R4)
                Pi = 0.5 * (Pi + Pi.T)
                eps = error_bound(B, res.X, res.theta)
                p = int(np.sum(pos))
                if s > 0:
                    self.last_pos, self.last_neg = p, n - p
                else:
                    self.last_neg, self.last_pos = p, n - p
                keep = self._keep(res.theta, res.m)
                self.X = res.X[:, :keep].copy()
                self.block_side = mode
                info.update(status=res.status, iters=res.iters, m=res.m, npos=p, err_bound=eps,
                            trace=res.trace, expansions=res.expansions, a_passes=res.a_passes, a_cols=res.a_cols,
                            cold=cold, theta=res.theta, r=res.r, side=mode)
                return Pi, info
        # DIRECT: full eigendecomposition (PAPER.md:505 'otherwise', R18)
        w, V, _ = jacobi_eig(A)
        pos = w > 0
        Pi = (V[:, pos] * w[pos]) @ V[:, pos].T
        Pi = 0.5 * (Pi + Pi.T)
        z = 1e-9 * (1.0 + np.linalg.norm(A))
        self.last_pos = int(np.sum(w > z))
        self.last_neg = int(np.sum(w < -z))
        # seed the warm block of the side the next call will use
        nxt = self.select_mode()
        if nxt in (POS, NEG):
            s = 1.0 if nxt == POS else -1.0
            order = np.argsort(-(s * w), kind="stable")
            th = (s * w)[order]
            keep = self._keep(th, n)
            self.X = V[:, order[:keep]].copy()
            self.block_side = nxt
        else:
            self.X = None
            self.block_side = 0
        info.update(status=OK, iters=0, npos=int(np.sum(pos)), err_bound=direct_bound(A, V, w), side=DIRECT, w=w)
        return Pi, info
