"""f4: one-CTA warm LOBPCG per tiny block (psdproj_project_tiny_lobpcg) on BO-like
blocks (rank-one PSD parts; workloads.generators.BO) against the oracle's exact
projection (O-EXACT): parity at the BJ threshold, bound dominance, warm < cold, and the exact-path
hand-off for blocks that outgrow the one-CTA capacity."""
import numpy as np
import pytest
import torch

from oracle.exact import project_exact
from workloads.generators import BO, haar_q, planted

pytestmark = pytest.mark.gpu


def test_tiny_lobpcg_bo_sequence(api):
    cfg = BO(count=48, lo=8, hi=100)
    ids = range(cfg.count)
    mats = [planted(*cfg.block(i)) for i in ids]
    batch = api.TinyLobpcgBatch(cfg.sizes, seed=7)
    its = []
    for rnd in range(3):
        outs, res = batch.project([torch.from_numpy(A).cuda() for A in mats], 1e-10)
        its.append(np.mean(res["iters"]))
        for i, A in enumerate(mats):
            Pg = outs[i].cpu().numpy()
            err = np.linalg.norm(Pg - project_exact(A))
            nA = np.linalg.norm(A)
            assert res["status"][i] in (0, 3), (rnd, i, res["status"][i])
            assert err / nA <= 1e-9, (rnd, i, cfg.sizes[i], err / nA)
            assert np.array_equal(Pg, Pg.T)
            assert res["npos"][i] == 1
            if res["status"][i] == 0:
                assert res["bound"][i] >= err, (rnd, i, err, res["bound"][i])
        mats = [A + cfg.drift(i, rnd) for A, i in zip(mats, ids)]
    assert its[1] < its[0] and its[2] < its[0], its     # warm rounds need fewer iterations than cold


def test_tiny_lobpcg_hands_wide_blocks_to_exact_path(api):
    """A block with 12 positive eigenvalues outgrows the 8-column one-CTA block: the exact path
    projects it (status 3); a tiny n (= 4) goes there directly."""
    rng = np.random.default_rng(3)
    wide = planted(haar_q(rng, 60), np.concatenate([rng.uniform(1, 3, 12), rng.uniform(-3, -1, 48)]))
    small = planted(haar_q(rng, 4), np.array([2.0, -1.0, -2.0, -3.0]))
    ok = planted(haar_q(rng, 40), np.concatenate([[5.0], rng.uniform(-3, -0.5, 39)]))
    mats = [wide, small, ok]
    batch = api.TinyLobpcgBatch([A.shape[0] for A in mats])
    outs, res = batch.project([torch.from_numpy(A).cuda() for A in mats], 1e-10)
    assert res["status"][0] == 3 and res["status"][1] == 3 and res["status"][2] == 0, res
    assert res["npos"] == [12, 1, 1]
    for A, P in zip(mats, outs):
        assert np.linalg.norm(P.cpu().numpy() - project_exact(A)) <= 1e-11 * np.linalg.norm(A)
