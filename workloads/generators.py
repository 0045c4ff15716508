"""Seeded synthetic workloads (BASELINE.json configs; recipes in DESIGN.md §4).

Conventions:
  * planted eigenbasis Q: Q, R = qr(standard_normal((n, n))); Q *= sign(diag(R))
  * A_0 = Q diag(lam) Q^T, symmetrised (A + A^T)/2 (R23)
  * additive drift (C1, C2, C3, C4): A_{t+1} = A_t + eps_t * sym(G_t), G_t i.i.d. N(0,1) from
    default_rng([seed, t]) (R29: sym(G) = (G + G^T)/2)
  * C3-R (spectrum-preserving, R30): Q_{t+1} = qr_signfix(Cay(eps_t K_t) Q_t),
    K_t = (G_t - G_t^T) / (2 sqrt(n)), Cay(K) = (I - K/2)^{-1} (I + K/2), eps_t = 1e-2 / t,
    A_t = Q_t diag(lam) Q_t^T -- exactly 5% positive at every step.
No projection / eigensolver arithmetic lives here.
"""
import math
from dataclasses import dataclass

import numpy as np


def sym(M):
    return 0.5 * (M + M.T)


def haar_q(rng, n):
    Q, R = np.linalg.qr(rng.standard_normal((n, n)))
    Q *= np.sign(np.diag(R))
    return Q


def planted(Q, lam):
    return sym((Q * lam) @ Q.T)


@dataclass
class Config:
    name: str
    n: int
    seed: int
    steps: int
    tol: float
    kind: str  # 'additive' | 'rotation'

    def spectrum(self, rng):
        raise NotImplementedError

    def eps(self, t):
        raise NotImplementedError


class _C1(Config):
    def spectrum(self, rng):
        return np.concatenate([rng.uniform(0.1, 10, 10), rng.uniform(-10, -0.1, self.n - 10)])

    def eps(self, t):
        return 1e-3


class _C2(Config):
    clustered = False

    def spectrum(self, rng):
        n = self.n
        lam = np.concatenate([rng.uniform(0.01, 100, 40), rng.uniform(-100, -0.01, n - 40)])
        if self.clustered:  # R31: first 20 negatives -> U[-1e-6, 1e-6]
            lam[40:60] = rng.uniform(-1e-6, 1e-6, 20)
        return lam

    def eps(self, t):
        return 1e-4


class _C2CL(_C2):
    clustered = True


class _C3(Config):
    """n=4000, 5% positive log-uniform [1e-3, 1e2], negatives mirrored (BASELINE configs[2])."""

    def spectrum(self, rng):
        n = self.n
        p = int(round(0.05 * n))
        return np.concatenate([10.0 ** rng.uniform(-3, 2, p), -(10.0 ** rng.uniform(-3, 2, n - p))])

    def eps(self, t):
        return 1e-2 / t


def C1(n=200):
    return _C1("C1", n, 101, 50, 1e-10, "additive")


def C2(n=1000):
    return _C2("C2", n, 201, 200, 1e-8, "additive")


def C2CL(n=1000):
    return _C2CL("C2-cl", n, 202, 200, 1e-8, "additive")


def C3(n=4000):
    return _C3("C3", n, 301, 500, 1e-7, "additive")


def C3R(n=4000):
    return _C3("C3-R", n, 302, 500, 1e-7, "rotation")


def initial(cfg):
    rng = np.random.default_rng(cfg.seed)
    lam = cfg.spectrum(rng)
    Q = haar_q(rng, cfg.n)
    return Q, lam


def drift_sequence(cfg, steps=None, start=None):
    """Yields (t, A_t, extra) for t = 0..steps-1 of an additive-drift config.
    extra = (Q, lam) at t = 0 (A_0 planted), else None."""
    steps = cfg.steps if steps is None else steps
    Q, lam = initial(cfg) if start is None else start
    A = planted(Q, lam)
    for t in range(steps):
        yield t, A, ((Q, lam) if t == 0 else None)
        G = np.random.default_rng([cfg.seed, t]).standard_normal((cfg.n, cfg.n))
        A = A + cfg.eps(t + 1) * sym(G)


def rotation_sequence(cfg, steps=None, device=None, start=None, t0=0):
    """Yields (t, A_t, Q_t, lam) for the spectrum-preserving C3-R drift. With device (a torch
    device string) the Cayley step and products run in torch float64 there (same recipe).
    start = (Q, lam) with t0: continue from that state with the drift of steps t0, t0 + 1, ...
    (eps(t + 1) and the seed stream [seed, t]); the Cayley rotation is Haar-invariant, so a state
    reached after t0 steps and any other orthogonal Q are statistically the same start."""
    steps = cfg.steps if steps is None else steps
    Q, lam = initial(cfg) if start is None else start
    n = cfg.n
    if device is None:
        for t in range(t0, t0 + steps):
            yield t, planted(Q, lam), Q, lam
            G = np.random.default_rng([cfg.seed, t]).standard_normal((n, n))
            K = (G - G.T) / (2.0 * math.sqrt(n)) * cfg.eps(t + 1)
            I = np.eye(n)
            Y = np.linalg.solve(I - 0.5 * K, (I + 0.5 * K) @ Q)
            Q, R = np.linalg.qr(Y)
            Q *= np.sign(np.diag(R))
    else:
        import torch

        Qd = torch.as_tensor(Q, device=device)
        lamd = torch.as_tensor(lam, device=device)
        I = torch.eye(n, dtype=torch.float64, device=device)
        for t in range(t0, t0 + steps):
            A = (Qd * lamd) @ Qd.T
            A = 0.5 * (A + A.T)
            yield t, A, Qd, lamd
            G = torch.as_tensor(np.random.default_rng([cfg.seed, t]).standard_normal((n, n)), device=device)
            K = (G - G.T) / (2.0 * math.sqrt(n)) * cfg.eps(t + 1)
            Y = torch.linalg.solve(I - 0.5 * K, (I + 0.5 * K) @ Qd)
            Qd, R = torch.linalg.qr(Y)
            Qd = Qd * torch.sign(torch.diagonal(R))


class C4:
    """512 independent blocks, n_i ~ U{50,100,200,400}, positive fraction f_i ~ U[0.05,0.5],
    p_i = max(1, round(f_i n_i)); positives U(0,1], negatives U[-1,0); drift 1e-3 sym(G) per
    round (R32), tol 1e-8 (R32)."""

    name = "C4"
    seed = 401
    tol = 1e-8
    rounds = 100

    def __init__(self, count=512, sizes=(50, 100, 200, 400)):
        rng = np.random.default_rng(self.seed)
        self.count = count
        self.sizes = [int(x) for x in rng.choice(sizes, count)]
        self.fracs = rng.uniform(0.05, 0.5, count)
        self.npos = [max(1, int(round(f * n))) for f, n in zip(self.fracs, self.sizes)]

    def block(self, i):
        n, p = self.sizes[i], self.npos[i]
        rng = np.random.default_rng([self.seed, i])
        lam = np.concatenate([1.0 - rng.uniform(0.0, 1.0, p), -rng.uniform(0.0, 1.0, n - p)])
        Q = haar_q(rng, n)
        return Q, lam

    def drift(self, i, r):
        n = self.sizes[i]
        return 1e-3 * sym(np.random.default_rng([self.seed, i, r]).standard_normal((n, n)))


def c4_blocks(count=512):
    return C4(count)


def maxcut_graph(n=2000, p_edge=0.01, seed=501):
    """C5: Erdos-Renyi graph, weights +-1 (BASELINE configs[4]); returns the Laplacian
    L = diag(W 1) - W (dense fp64)."""
    rng = np.random.default_rng(seed)
    iu = np.triu_indices(n, 1)
    mask = rng.uniform(size=iu[0].size) < p_edge
    w = np.where(rng.uniform(size=int(mask.sum())) < 0.5, -1.0, 1.0)
    W = np.zeros((n, n))
    W[iu[0][mask], iu[1][mask]] = w
    W = W + W.T
    return np.diag(W.sum(axis=1)) - W


class BO:
    """f4 stand-in for the Bayesian-optimisation SDPs of PAPER.md:605-649 (their data are not in the
    container): `count` independent blocks, n_i ~ U{lo..hi}, a rank-one PSD part (one eigenvalue ~ U[1, 10],
    P:647 "rank-one solutions") and the rest ~ U[-5, -0.1], planted Q_i; each round drifts every block by
    1e-3 sym(G) (as C4, R32)."""

    seed = 601
    tol = 1e-10

    def __init__(self, count=4096, lo=8, hi=100):
        rng = np.random.default_rng(self.seed)
        self.count = count
        self.sizes = [int(x) for x in rng.integers(lo, hi + 1, count)]

    def block(self, i):
        n = self.sizes[i]
        rng = np.random.default_rng([self.seed, i])
        lam = np.concatenate([rng.uniform(1.0, 10.0, 1), -rng.uniform(0.1, 5.0, n - 1)])
        return haar_q(rng, n), lam

    def drift(self, i, r):
        n = self.sizes[i]
        return 1e-3 * sym(np.random.default_rng([self.seed, i, r]).standard_normal((n, n)))
