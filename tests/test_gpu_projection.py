"""GPU projection parity (C ABI) against the oracle's exact projection (O-EXACT)."""
import numpy as np
import pytest
import torch

from oracle.exact import project_exact
from workloads.generators import C1, drift_sequence, haar_q, planted

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_c1_sequence_parity(api):
    cfg = C1()
    ctx = api.Context(cfg.n, seed=7)
    for t, A, _ in drift_sequence(cfg, steps=6):
        Pi, info = ctx.project(_dev(A), 1e-10)
        Pe = project_exact(A)
        Pg = Pi.cpu().numpy()
        err = np.linalg.norm(Pg - Pe)
        assert info["status"] in (0, 1)
        assert err / np.linalg.norm(A) <= 1e-9, (t, err, info)
        assert info["err_bound"] >= err, (t, err, info["err_bound"])
        assert np.array_equal(Pg, Pg.T)
        assert info["npos"] == 10


@pytest.mark.parametrize("n,p,side", [(60, 5, 1), (60, 55, -1), (120, 10, 0), (300, 12, 0), (300, 280, 0)])
def test_planted_parity(api, n, p, side):
    rng = np.random.default_rng(n * 7 + p)
    lam = np.concatenate([rng.uniform(0.1, 5, p), rng.uniform(-5, -0.1, n - p)])
    Q = haar_q(rng, n)
    A = planted(Q, lam)
    Pstar = (Q * np.maximum(lam, 0)) @ Q.T
    ctx = api.Context(n, side=side, seed=3)
    for call in range(2):
        Pi, info = ctx.project(_dev(A), 1e-10)
        err = np.linalg.norm(Pi.cpu().numpy() - Pstar)
        assert err / np.linalg.norm(A) <= 1e-9, (call, err, info)
        assert info["err_bound"] >= err - 1e-12 * np.linalg.norm(A)
