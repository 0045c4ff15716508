"""Synthetic workloads (workloads/generators.py): shapes, seeds, and the planted spectra the
configs promise (BASELINE.json configs)."""
import numpy as np

from workloads.generators import C1, C2CL, C3, C3R, C4, drift_sequence, maxcut_graph, rotation_sequence


def test_c1_spectrum_and_drift():
    cfg = C1()
    seq = drift_sequence(cfg, steps=3)
    t, A0, (Q, lam) = next(seq)
    assert A0.shape == (200, 200) and np.array_equal(A0, A0.T)
    assert np.sum(lam > 0) == 10 and np.all((lam[:10] >= 0.1) & (lam[:10] <= 10))
    assert np.linalg.norm(Q.T @ Q - np.eye(200)) < 1e-12
    t, A1, _ = next(seq)
    G = np.random.default_rng([101, 0]).standard_normal((200, 200))
    assert np.allclose(A1 - A0, 1e-3 * 0.5 * (G + G.T), atol=1e-15)


def test_c2_clustered_variant():
    cfg = C2CL(n=200)
    from workloads.generators import initial
    Q, lam = initial(cfg)
    assert np.all(np.abs(lam[40:60]) <= 1e-6)


def test_c3r_keeps_five_percent():
    cfg = C3R(n=200)
    for t, A, Q, lam in rotation_sequence(cfg, steps=3):
        assert np.sum(lam > 0) == 10
        assert np.linalg.norm(Q.T @ Q - np.eye(200)) < 1e-12
        assert np.linalg.norm(A - (Q * lam) @ Q.T) < 1e-12 * np.linalg.norm(A)
    assert np.all(np.abs(lam) >= 1e-3 * (1 - 1e-12)) and np.all(np.abs(lam) <= 1e2)


def test_c3r_continue_from_state():
    """rotation_sequence(start=(Q_t, lam), t0=t) continues the same sequence (bench.py's late-sequence
    companion applies the drift of t = 100.. from the last timed state)."""
    cfg = C3R(n=120)
    full = list(rotation_sequence(cfg, steps=5))
    cont = list(rotation_sequence(cfg, steps=3, start=(full[2][2], full[2][3]), t0=2))
    assert [c[0] for c in cont] == [2, 3, 4]
    for c, f in zip(cont, full[2:]):
        assert np.array_equal(c[1], f[1])
    # the drift of step t rotates by ~eps(t + 1): a late start moves the matrix less
    late = list(rotation_sequence(cfg, steps=2, start=(full[2][2], full[2][3]), t0=99))
    d_late = np.linalg.norm(late[1][1] - late[0][1])
    d_early = np.linalg.norm(full[3][1] - full[2][1])
    assert d_late < d_early * (3.0 / 100.0) * 1.5


def test_c3_literal_loses_five_percent():
    """F4 of SURVEY.md: the literal additive drift of configs[2] smears the near-zero spectrum
    (measured at n = 400 here: positive count grows well beyond 5%)."""
    cfg = C3(n=400)
    seq = drift_sequence(cfg, steps=2)
    _, A0, _ = next(seq)
    _, A1, _ = next(seq)
    assert np.sum(np.linalg.eigvalsh(A0) > 0) == 20
    assert np.sum(np.linalg.eigvalsh(A1) > 0) > 40


def test_c4_blocks():
    c4 = C4(count=16)
    assert set(c4.sizes) <= {50, 100, 200, 400}
    Q, lam = c4.block(3)
    assert len(lam) == c4.sizes[3] and np.sum(lam > 0) == c4.npos[3]
    assert np.all(lam[: c4.npos[3]] > 0) and np.all(lam[c4.npos[3]:] <= 0)


def test_maxcut_laplacian():
    L = maxcut_graph(n=300, p_edge=0.05)
    assert np.array_equal(L, L.T)
    assert np.allclose(L.sum(axis=1), 0)
