"""GPU-vs-oracle parity through the C ABI, round 2 additions:

  * C2 and C2-cl (BASELINE configs[1], n = 1000): all 200 warm steps through the library at the
    parity tolerance 1e-10; every 10th step against O-EXACT fingerprints written by
    tools/make_golden_c2.py from oracle/ only (tests/golden/c2_oracle.npz: the oracle's cyclic
    Jacobi needs ~1 min per n = 1000 matrix). Checks: Pi (a Gaussian-probe estimate of the
    Frobenius error and a deterministic lower bound of it that the reported bound must dominate),
    Ritz values through psdproj_get_ritz in the R34 form, positive counts.
  * Ritz-value parity (north star: "eigenvalues within 1e-10 relative", reading R34) on planted
    spectra against the oracle's Jacobi eigenvalues.
  * psdproj_reset on a live context: the next call is cold and still oracle-matching.
"""
import os

import numpy as np
import pytest
import torch

from oracle.exact import eig, project_exact
from workloads.generators import C1, C2, C2CL, drift_sequence, haar_q, planted

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c2_oracle.npz")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _r34_ok(theta, lam, a2):
    """R34: |theta_i - lambda_i| <= 1e-10 max(|lambda_i|, 1e-3 ||A||_2), matched by descending sort."""
    return np.abs(theta - lam) <= 1e-10 * np.maximum(np.abs(lam), 1e-3 * a2)


@pytest.mark.parametrize("which", ["C2", "C2-cl"])
def test_c2_sequence_every_10th_step(api, which):
    cfg = C2() if which == "C2" else C2CL()
    gold = np.load(GOLD)
    key0 = cfg.name.replace("-", "")
    Z = np.random.default_rng(20191206).standard_normal((cfg.n, 4))
    z2 = np.linalg.norm(Z, 2)
    ctx = api.Context(cfg.n, params=api.default_params(seed=202, max_iter=4000))
    checked = capped = 0
    for t, A, _ in drift_sequence(cfg, steps=cfg.steps):
        Pi, info = ctx.project(_dev(A), 1e-10)
        assert info["status"] in (0, 1), (t, info["iters"])
        capped += info["status"] == 1   # a cluster member crossing zero can stall a step at 1e-10
        if t % 10:
            continue
        key = f"{key0}_{t}"
        nA = float(gold[f"af_{key}"])
        assert abs(nA - np.linalg.norm(A)) <= 1e-12 * nA          # same seeded input
        EZ = Pi.cpu().numpy() @ Z - gold[f"piz_{key}"]
        ez = np.linalg.norm(EZ)
        assert ez / 2.0 <= 1e-9 * nA, (t, ez / 2.0 / nA)              # E||EZ||^2 = 4 ||E||_F^2
        assert info["err_bound"] >= ez / z2, (t, info["err_bound"], ez / z2)   # ||E||_F >= ||EZ||_F / ||Z||_2
        w = gold[f"w_{key}"]
        a2 = float(np.max(np.abs(w)))
        z = 1e-9 * (1.0 + nA)                                        # zero band for counts (R19)
        side = info["side"]
        lam = w if side == 1 else -w[::-1]                           # descending on the computed side
        theta = api_ritz = ctx.get_ritz().numpy()
        npos = int(np.sum(theta > 0))
        assert npos == info["npos"]
        assert int(np.sum(lam > z)) <= npos <= int(np.sum(lam > -z)), (t, npos)
        k = int(np.sum(lam > z))                                    # pairs clear of the zero band
        assert np.all(_r34_ok(theta[:k], lam[:k], a2)), (t, np.max(np.abs(theta[:k] - lam[:k])))
        assert np.all(np.abs(api_ritz[k:npos]) <= z)
        checked += 1
    assert checked == 20
    assert capped <= 5, capped


@pytest.mark.parametrize("n,p,scale", [(120, 9, 1.0), (300, 25, 100.0), (500, 12, 1e-3)])
def test_ritz_values_parity(api, n, p, scale):
    """Computed-side Ritz values (psdproj_get_ritz) against the oracle's Jacobi eigenvalues of A,
    R34 form, with count equality; spectra with a near-zero positive tail and a wide range."""
    rng = np.random.default_rng(n + p)
    lam = scale * np.concatenate([10.0 ** rng.uniform(-3, 1, p), -(10.0 ** rng.uniform(-3, 1, n - p))])
    A = planted(haar_q(rng, n), lam)
    w, _ = eig(A)                       # oracle eigenvalues (cyclic Jacobi), ascending
    w = w[::-1]
    ctx = api.Context(n, params=api.default_params(seed=5, side=1, max_iter=6000))
    for call in range(2):
        Pi, info = ctx.project(_dev(A), 1e-10 * scale)
        assert info["status"] == 0
        theta = ctx.get_ritz().numpy()
        npos = int(np.sum(theta > 0))
        assert npos == p == info["npos"]
        a2 = float(np.max(np.abs(w)))
        assert np.all(_r34_ok(theta[:p], w[:p], a2)), np.max(np.abs(theta[:p] - w[:p]))
        vals, vecs = ctx.get_ritz(with_vectors=True)
        V = vecs.cpu().numpy()[:, :p]
        assert np.linalg.norm(V.T @ V - np.eye(p)) <= 1e-12 * p
        R = A @ V - V * vals.numpy()[:p]
        assert np.all(np.linalg.norm(R, axis=0) <= 1e-10 * scale * 1.0001 + 1e-13 * np.linalg.norm(A))


def test_reset_makes_next_call_cold(api):
    """psdproj_reset on a live context: the warm block is dropped, the next call starts cold
    (Philox block, m0 = ceil(0.1 n), R28) and is still oracle-matching; warm iterations < cold."""
    cfg = C1()
    ctx = api.Context(cfg.n, params=api.default_params(seed=17))
    seq = list(drift_sequence(cfg, steps=4))
    iters = {}
    for t, A, _ in seq[:3]:
        _, info = ctx.project(_dev(A), 1e-10)
        iters[t] = info
    assert iters[0]["cold"] == 1 and iters[1]["cold"] == 0 and iters[2]["cold"] == 0
    ctx.reset()
    assert ctx.get_ritz().numel() == 0
    t, A, _ = seq[3]
    Pi, info = ctx.project(_dev(A), 1e-10)
    assert info["cold"] == 1
    err = np.linalg.norm(Pi.cpu().numpy() - project_exact(A))
    assert err / np.linalg.norm(A) <= 1e-9 and info["err_bound"] >= err
    assert iters[2]["iters"] < info["iters"]
