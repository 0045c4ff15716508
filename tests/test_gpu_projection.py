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
    """BASELINE configs[0], all 50 steps of the warm sequence against O-EXACT."""
    cfg = C1()
    ctx = api.Context(cfg.n, seed=7)
    for t, A, _ in drift_sequence(cfg, steps=cfg.steps):
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
        assert info["err_bound"] >= err, (call, err, info["err_bound"])


# ---------------------------------------------------------------- edge cases
@pytest.mark.parametrize("case", ["n1_pos", "n1_neg", "n2_diag", "zero", "minus_identity", "psd", "rank1",
                                  "n4_one_pos", "k4_laplacian"])
def test_edge_cases(api, case):
    rng = np.random.default_rng(11)
    if case == "n1_pos":
        A, expect = np.array([[2.5]]), np.array([[2.5]])
    elif case == "n1_neg":
        A, expect = np.array([[-3.0]]), np.zeros((1, 1))
    elif case == "n2_diag":
        A, expect = np.diag([1.0, -1.0]), np.diag([1.0, 0.0])
    elif case == "zero":
        A = np.zeros((40, 40))
        expect = A.copy()
    elif case == "minus_identity":
        A, expect = -np.eye(50), np.zeros((50, 50))
    elif case == "psd":
        M = rng.standard_normal((30, 8))
        A = M @ M.T
        expect = A.copy()
    elif case == "n4_one_pos":  # cold block of one column locks at once with no guard column (R8)
        Q = np.linalg.qr(rng.standard_normal((4, 4)))[0]
        A = (Q * np.array([3.0, -1.0, -2.0, -3.0])) @ Q.T
        A = 0.5 * (A + A.T)
        expect = project_exact(A)
    elif case == "k4_laplacian":  # repeated eigenvalues {0, 4, 4, 4} shifted: {-1, 3, 3, 3}
        A = 4.0 * np.eye(4) - np.ones((4, 4)) - np.eye(4)
        expect = project_exact(A)
    else:
        v = rng.standard_normal(64)
        A = np.outer(v, v) - 0.5 * np.eye(64)
        expect = project_exact(A)
    n = A.shape[0]
    ctx = api.Context(n, seed=5)
    for call in range(2):  # cold, then warm
        Pi, info = ctx.project(_dev(A), 1e-10)
        err = np.linalg.norm(Pi.cpu().numpy() - expect)
        assert info["status"] in (0, 1), info
        assert err <= 1e-9 * max(1.0, np.linalg.norm(A)), (case, call, err, info)
        assert info["err_bound"] >= err, (case, call, err, info["err_bound"])


def test_nonfinite_input_is_rejected(api):
    A = np.eye(20)
    A[3, 7] = A[7, 3] = np.nan
    ctx = api.Context(20)
    with pytest.raises(api.PsdprojError if hasattr(api, "PsdprojError") else Exception) as ei:
        ctx.project(_dev(A), 1e-8)
    assert "-2" in str(ei.value) or "nan" in str(ei.value).lower()


def test_direct_path_mixed_spectrum(api):
    """Half positive: the one-third rule takes the DIRECT eigensolver."""
    rng = np.random.default_rng(4)
    n = 180
    lam = rng.uniform(-1, 1, n)
    A = planted(haar_q(rng, n), lam)
    ctx = api.Context(n, seed=2)
    ctx.project(_dev(A), 1e-10)      # cold call learns the counts
    Pi, info = ctx.project(_dev(A), 1e-10)
    assert info["side"] == 2
    Pstar = project_exact(A)
    err = np.linalg.norm(Pi.cpu().numpy() - Pstar)
    assert err <= 1e-11 * np.linalg.norm(A)
    # R53: a real bound on the DIRECT path (explicit residuals of all n pairs), at the rounding level
    assert err <= info["err_bound"] <= 200 * n * 2.0 ** -53 * np.linalg.norm(A), (err, info["err_bound"])


def test_host_io_matches_device(api):
    cfg = C1()
    seq = drift_sequence(cfg, steps=2)
    _, A0, _ = next(seq)
    _, A1, _ = next(seq)
    dctx = api.Context(cfg.n, params=api.default_params(seed=9))
    hctx = api.Context(cfg.n, params=api.default_params(seed=9, host_io=1))
    for A in (A0, A1):
        Pd, _ = dctx.project(_dev(A), 1e-10)
        Ph, info = hctx.project_host(torch.from_numpy(A.copy()), 1e-10)
        assert np.array_equal(Pd.cpu().numpy(), Ph.numpy())


def test_determinism_bitwise(api):
    """Fixed-order reductions (R25): same inputs and seed -> bitwise identical Pi and info."""
    rng = np.random.default_rng(8)
    lam = np.concatenate([rng.uniform(0.1, 3, 15), rng.uniform(-3, -0.1, 285)])
    A = planted(haar_q(rng, 300), lam)
    outs = []
    for _ in range(2):
        ctx = api.Context(300, seed=21)
        Pi, info = ctx.project(_dev(A), 1e-9)
        outs.append((Pi.cpu().numpy(), info["iters"], info["err_bound"]))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1:] == outs[1][1:]


def test_c4_batched_parity(api):
    """BASELINE configs[3] blocks through psdproj_project_batched (threaded, one stream per worker):
    every block matches the oracle's exact projection and its bound dominates the error."""
    from workloads.generators import C4
    cfg = C4(24)
    ids = list(range(24))
    mats = [planted(*cfg.block(i)) for i in ids]
    ctxs = [api.Context(cfg.sizes[i], params=api.default_params(seed=3, ctx_id=i)) for i in ids]
    for rnd in range(2):
        outs, infos = api.project_batched(ctxs, [_dev(A) for A in mats], [1e-10] * len(ids))
        for k, i in enumerate(ids):
            Pe = project_exact(mats[k])
            err = np.linalg.norm(outs[k].cpu().numpy() - Pe)
            nA = np.linalg.norm(mats[k])
            assert infos[k]["status"] in (0, 1), (i, infos[k])
            assert err / nA <= 1e-9, (rnd, i, cfg.sizes[i], err / nA, infos[k]["side"])
            assert infos[k]["err_bound"] >= err, (rnd, i, err, infos[k]["err_bound"])
        mats = [A + cfg.drift(i, rnd) for A, i in zip(mats, ids)]


def test_c3r_reduced_sequence(api):
    """C3-R at n = 1000 (configs[2] spectrum; closed-form Pi*_t = Q_t max(L, 0) Q_t^T), every step of
    a 26-step warm run, run to convergence (status OK): the bound dominates the true error on every
    call (no allowance) and the error is within the config's accuracy; the last (warm) step at the
    parity tolerance 1e-10 meets the BJ threshold 1e-9."""
    from workloads.generators import C3R, rotation_sequence
    cfg = C3R(1000)
    ctx = api.Context(cfg.n, params=api.default_params(seed=4, max_iter=6000))
    for t, A, Q, lam in rotation_sequence(cfg, steps=26, device="cuda"):
        tol = 1e-10 if t == 25 else cfg.tol
        Pi, info = ctx.project(A.contiguous(), tol)
        Pstar = (Q * torch.clamp(lam, min=0)) @ Q.T
        err = float(torch.linalg.norm(Pi - Pstar))
        nA = float(torch.linalg.norm(A))
        assert info["status"] == 0, (t, info["iters"])
        assert info["npos"] == 50                              # exactly 5% positive at every step
        assert info["err_bound"] >= err, (t, err, info["err_bound"])
        assert err / nA <= (1e-9 if tol == 1e-10 else 2e-9), (t, err / nA)


def test_full_size_full_matrix(api):
    """BASELINE's full size n = 4000 in the bench's launch configuration (C3-R, tol 1e-7, the bench's
    max_iter): the whole Pi against the closed form on the GPU, every call bound-verified."""
    from workloads.generators import C3R, rotation_sequence
    cfg = C3R(4000)
    ctx = api.Context(cfg.n, params=api.default_params(seed=1912, max_iter=4000, profile=0))
    for t, A, Q, lam in rotation_sequence(cfg, steps=3, device="cuda"):
        Pi, info = ctx.project(A.contiguous(), cfg.tol)
        Pstar = (Q * torch.clamp(lam, min=0)) @ Q.T
        err = float(torch.linalg.norm(Pi - Pstar))
        nA = float(torch.linalg.norm(A))
        assert info["status"] == 0, (t, info)
        assert info["npos"] == 200
        assert info["err_bound"] >= err, (t, err, info["err_bound"])
        assert err / nA <= 2e-9 and info["err_bound"] / nA <= 2e-9, (t, err / nA, info["err_bound"] / nA)
        assert torch.equal(Pi, Pi.T)
        assert info["launches"] > 0


def test_row_sharded_single_rank_matches_unsharded(api):
    """Row-sharded mode (§8.e) with one rank: NCCL all-gathers / all-reduces on a 1-rank
    communicator; same iterates as the unsharded context, Pi = W W^T exactly symmetric, and the
    projection matches the oracle."""
    cfg = C1()
    uid = api.nccl_uid()
    sh = api.ShardedContext(cfg.n, 0, cfg.n, uid, 0, 1, params=api.default_params(seed=13))
    un = api.Context(cfg.n, params=api.default_params(seed=13))
    for t, A, _ in drift_sequence(cfg, steps=3):
        Ad = _dev(A)
        Ps, info_s = sh.project(api.colmajor_copy(Ad), 1e-10)
        Pu, info_u = un.project(Ad, 1e-10)
        Ps = Ps.cpu().numpy()
        assert info_s["iters"] == info_u["iters"] and info_s["npos"] == info_u["npos"]
        assert np.array_equal(Ps, Ps.T)
        assert np.linalg.norm(Ps - Pu.cpu().numpy()) <= 1e-12 * np.linalg.norm(A)
        assert np.linalg.norm(Ps - project_exact(A)) / np.linalg.norm(A) <= 1e-9
    sh.close()


@pytest.mark.parametrize("locking", [1, 2])
def test_locking_modes_parity(api, locking):
    """Soft (BLOPEX active mask) and hard locking (R35) reach the same projection."""
    rng = np.random.default_rng(21)
    n, p = 240, 14
    lam = np.concatenate([rng.uniform(0.2, 4, p), rng.uniform(-4, -0.2, n - p)])
    Q = haar_q(rng, n)
    A = planted(Q, lam)
    Pstar = (Q * np.maximum(lam, 0)) @ Q.T
    ctx = api.Context(n, params=api.default_params(seed=5, locking=locking))
    Pi, info = ctx.project(_dev(A), 1e-10)
    err = np.linalg.norm(Pi.cpu().numpy() - Pstar)
    assert info["status"] == 0, info
    assert err / np.linalg.norm(A) <= 1e-9
    assert info["err_bound"] >= err, (err, info["err_bound"])
    if locking == 1:
        assert info["locked"] == 0


def test_random_expansion_path(api):
    """A cold block narrower than the positive eigenspace saturates and is widened by random
    Philox columns (Alg. 3 line 8; R8-R11) until a guard appears."""
    rng = np.random.default_rng(22)
    n, p = 300, 40
    lam = np.concatenate([rng.uniform(0.5, 5, p), rng.uniform(-5, -0.5, n - p)])
    Q = haar_q(rng, n)
    A = planted(Q, lam)
    Pstar = (Q * np.maximum(lam, 0)) @ Q.T
    ctx = api.Context(n, params=api.default_params(seed=6, m0=8, expand_q=12, side=1))
    Pi, info = ctx.project(_dev(A), 1e-10)
    assert info["expansions"] >= 1 and info["npos"] == p, info
    assert np.linalg.norm(Pi.cpu().numpy() - Pstar) / np.linalg.norm(A) <= 1e-9


@pytest.mark.parametrize("n,p", [(13, 3), (77, 9), (129, 100), (333, 21), (517, 60)])
def test_odd_sizes_parity(api, n, p):
    """Ragged orders (ld rounding, partial tiles in every kernel) on both sides of the one-third rule."""
    rng = np.random.default_rng(n + p)
    lam = np.concatenate([rng.uniform(0.05, 3, p), rng.uniform(-3, -0.05, n - p)])
    Q = haar_q(rng, n)
    A = planted(Q, lam)
    Pstar = (Q * np.maximum(lam, 0)) @ Q.T
    ctx = api.Context(n, seed=8)
    for call in range(3):
        Pi, info = ctx.project(_dev(A), 1e-10)
        err = np.linalg.norm(Pi.cpu().numpy() - Pstar)
        assert info["status"] in (0, 1)
        assert err / np.linalg.norm(A) <= 1e-9, (call, err, info["side"], info["iters"])
        assert info["err_bound"] >= err, (call, err, info["err_bound"])


def test_tiny_batched_parity(api):
    """f4: many tiny blocks in one launch (one CTA each, exact one-CTA Jacobi): every block equals
    the oracle's exact projection, exactly symmetric, with the right positive count."""
    rng = np.random.default_rng(31)
    sizes = [1, 2, 3, 7, 16, 33, 64, 100, 112, 5, 8, 40]
    mats, expect = [], []
    for k, n in enumerate(sizes):
        kind = k % 4
        if kind == 0:
            A = rng.standard_normal((n, n))
            A = 0.5 * (A + A.T)
        elif kind == 1:  # PSD (rank deficient)
            M = rng.standard_normal((n, max(1, n // 3)))
            A = M @ M.T
        elif kind == 2:  # NSD
            M = rng.standard_normal((n, n))
            A = -(M @ M.T)
        else:            # planted spectrum with a near-zero cluster
            lam = np.concatenate([rng.uniform(-3, 3, n - n // 4), rng.uniform(-1e-10, 1e-10, n // 4)])
            A = planted(haar_q(rng, n), lam)
        mats.append(A)
        expect.append(project_exact(A))
    outs, npos = api.project_tiny_batched([_dev(A) for A in mats])
    for A, P, E, c in zip(mats, outs, expect, npos):
        Pg = P.cpu().numpy()
        assert np.linalg.norm(Pg - E) <= 1e-12 * max(1.0, np.linalg.norm(A)), A.shape
        assert np.array_equal(Pg, Pg.T)
        assert c == int(np.sum(np.linalg.eigvalsh(A) > 0)) or abs(np.sort(np.abs(np.linalg.eigvalsh(A)))[0]) < 1e-9


def test_tiny_batched_in_place_and_capacity(api):
    rng = np.random.default_rng(32)
    A = rng.standard_normal((20, 20))
    A = 0.5 * (A + A.T)
    E = project_exact(A)
    d = _dev(A)
    api.project_tiny_batched([d], outs=[d])  # Pi may alias A
    assert np.linalg.norm(d.cpu().numpy() - E) <= 1e-12 * np.linalg.norm(A)
    with pytest.raises(api.PsdprojError):
        api.project_tiny_batched([_dev(np.eye(113))])


@pytest.mark.parametrize("depth", [2])
def test_krylov_depth_parity(api, depth):
    """R57 (an extension of Alg. 3, off by default): block-Krylov trial subspaces reach the oracle's
    projection with every bound dominating, in fewer iterations than Alg. 3 on C3-R (n = 1000)."""
    from workloads.generators import C3R, rotation_sequence
    cfg = C3R(1000)
    its = {}
    for d in (1, depth):
        ctx = api.Context(cfg.n, params=api.default_params(seed=4, max_iter=6000, krylov_depth=d))
        tot = 0
        for t, A, Q, lam in rotation_sequence(cfg, steps=4, device="cuda"):
            Pi, info = ctx.project(A.contiguous(), cfg.tol)
            Pstar = (Q * torch.clamp(lam, min=0)) @ Q.T
            err = float(torch.linalg.norm(Pi - Pstar))
            nA = float(torch.linalg.norm(A))
            assert info["status"] == 0 and info["npos"] == 50, (d, t, info["iters"])
            assert info["err_bound"] >= err and err / nA <= 2e-9, (d, t, err / nA)
            if t > 0:
                tot += info["iters"]
        its[d] = tot
        ctx.close()
    assert its[depth] * 1.4 <= its[1], its


def test_krylov_max_active_parity(api):
    """R63: block-Krylov directions only while the active set is narrow (krylov_max_active). C3-R
    (n = 1000) warm sequence: closed-form projection, dominating bound, right positive count, fewer
    iterations than Alg. 3; a limit wider than any block equals R57 on every iteration bit for bit."""
    from workloads.generators import C3R, rotation_sequence
    cfg = C3R(1000)
    its, last = {}, {}
    for name, kw in (("alg3", dict(krylov_depth=1)), ("r57", dict(krylov_depth=2)),
                     ("wide", dict(krylov_depth=2, krylov_max_active=100000)),
                     ("mid", dict(krylov_depth=2, krylov_max_active=24))):
        ctx = api.Context(cfg.n, params=api.default_params(seed=4, max_iter=6000, **kw))
        tot = 0
        for t, A, Q, lam in rotation_sequence(cfg, steps=3, device="cuda"):
            Pi, info = ctx.project(A.contiguous(), cfg.tol)
            Pstar = (Q * torch.clamp(lam, min=0)) @ Q.T
            err = float(torch.linalg.norm(Pi - Pstar))
            nA = float(torch.linalg.norm(A))
            assert info["status"] == 0 and info["npos"] == 50, (name, t, info["iters"])
            assert info["err_bound"] >= err and err / nA <= 2e-9, (name, t, err / nA)
            if t > 0:
                tot += info["iters"]
        its[name] = tot
        last[name] = Pi.clone()
        ctx.close()
    assert torch.equal(last["wide"], last["r57"]) and its["wide"] == its["r57"], its
    assert its["r57"] <= its["mid"] < its["alg3"], its


def test_krylov_max_active_matches_oracle_iterates(api):
    """R63 against the oracle's LOBPCG with the same option (small planted problem, cold call): same
    iteration count and Ritz values to 1e-10 relative (R34 form)."""
    import oracle.lobpcg as L
    rng = np.random.default_rng(163)
    n, p = 240, 12
    lam = np.concatenate([10.0 ** rng.uniform(-1, 1, p), -(10.0 ** rng.uniform(-1, 1, n - p))])
    A = planted(haar_q(rng, n), lam)
    octx = L.Context(n, seed=9, ctx_id=0, krylov_depth=2, krylov_max_active=10)
    Po, io = octx.project(A, 1e-9)
    ctx = api.Context(n, params=api.default_params(seed=9, ctx_id=0, krylov_depth=2, krylov_max_active=10))
    Pi, info = ctx.project(torch.from_numpy(A).cuda(), 1e-9)
    th = np.sort(ctx.get_ritz().numpy())[::-1][:p]
    ctx.close()
    assert info["status"] == 0 and io["status"] == L.OK
    assert info["npos"] == io["npos"] == p
    assert abs(info["iters"] - io["iters"]) <= max(3, io["iters"] // 20), (info["iters"], io["iters"])
    top = np.sort(lam)[::-1][:p]
    assert np.max(np.abs(th - top) / np.maximum(np.abs(top), 1.0)) <= 1e-10
    assert np.linalg.norm(Pi.cpu().numpy() - Po) <= 1e-9 * np.linalg.norm(A)


def test_direct_path_large_order(api):
    """DIRECT on the tridiagonal eigensolver at n = 2000 (n <= EIG_MAX but > 3 m_max: the eigensolver
    scratch must be sized for n, not for the LOBPCG basis): a half-positive planted spectrum, cold
    call on the positive side expands past m_max and hands over to DIRECT (R18), then the one-third
    rule keeps it there; closed-form Pi*, the R53 bound dominates."""
    rng = np.random.default_rng(2000)
    n = 2000
    lam = rng.uniform(-1, 1, n)
    Q = haar_q(rng, n)
    A = planted(Q, lam)
    Pstar = (Q * np.maximum(lam, 0)) @ Q.T
    ctx = api.Context(n, seed=2)
    for call in range(2):
        Pi, info = ctx.project(_dev(A), 1e-10)
        err = np.linalg.norm(Pi.cpu().numpy() - Pstar)
        assert info["side"] == 2, info["side"]
        assert err <= 1e-11 * np.linalg.norm(A) and info["err_bound"] >= err, (call, err, info["err_bound"])


def test_c4_tiny_routing_parity(api):
    """C4 shard with the n <= 112 blocks routed through one launch of the one-CTA path (warm LOBPCG,
    exact hand-off) and the rest through contexts: every block matches the oracle's exact projection
    over two warm rounds; a LOBPCG-certified block's bound dominates its error."""
    import torch
    from paper_1912_02767_b200.multigpu import C4Shard
    from workloads.generators import C4
    cfg = C4(24)
    sh = C4Shard(cfg, list(range(24)), torch.device("cuda", 0))
    assert sh.small and sh.large
    paths = set()
    for rnd in range(2):
        infos = sh.project(1e-10)
        for k, i in enumerate(sh.ids):
            A = sh.mats[k].cpu().numpy()
            Pe = project_exact(A)
            err = np.linalg.norm(sh.outs[k].cpu().numpy() - Pe)
            nA = np.linalg.norm(A)
            assert infos[k]["status"] == 0, (rnd, i, infos[k])
            assert err / nA <= 1e-9, (rnd, i, cfg.sizes[i], err / nA, infos[k]["path"])
            if infos[k]["path"] in ("lobpcg", "tiny-lobpcg"):
                assert infos[k]["err_bound"] >= err, (rnd, i, err, infos[k])
            paths.add(infos[k]["path"])
        sh.drift()
    sh.close()
    assert "tiny-exact" in paths and "lobpcg" in paths, paths


def test_c4_direct_routing_parity(api):
    """C4 shard with direct_n = 200: the n = 200 contexts are created with side = DIRECT (the exact
    path a13), the n = 400 ones keep the one-third rule; every block matches the oracle's exact
    projection over two rounds, every bound dominates its error, and no n <= 200 context ran LOBPCG."""
    import torch
    from paper_1912_02767_b200.multigpu import C4Shard
    from workloads.generators import C4
    cfg = C4(24)
    sh = C4Shard(cfg, list(range(24)), torch.device("cuda", 0), direct_n=200)
    seen = {}
    for rnd in range(2):
        infos = sh.project(1e-10)
        for k, i in enumerate(sh.ids):
            A = sh.mats[k].cpu().numpy()
            err = np.linalg.norm(sh.outs[k].cpu().numpy() - project_exact(A))
            assert infos[k]["status"] == 0, (rnd, i, infos[k])
            assert err <= 1e-9 * np.linalg.norm(A), (rnd, i, cfg.sizes[i], infos[k]["path"])
            if infos[k]["path"] in ("lobpcg", "direct"):
                assert infos[k]["err_bound"] >= err, (rnd, i, err, infos[k])
            if 112 < cfg.sizes[i] <= 200:
                assert infos[k]["path"] == "direct", (rnd, i, infos[k])
            seen.setdefault(cfg.sizes[i], set()).add(infos[k]["path"])
        sh.drift()
    sh.close()
    assert 200 in seen and seen[200] == {"direct"}, seen
