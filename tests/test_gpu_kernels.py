"""GPU parity of the individual kernels (through the C ABI) against the oracle / definitions."""
import numpy as np
import pytest
import torch

from oracle.philox import gaussian_block, philox4x32_10

pytestmark = pytest.mark.gpu


def _cm(a):
    """numpy (r, c) -> column-major CUDA tensor view."""
    a = np.asarray(a, dtype=np.float64)
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda().T


@pytest.mark.parametrize("opA,opB", [(0, 0), (1, 0), (0, 1)])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (64, 64, 16), (131, 77, 203), (200, 40, 1000),
                                   (33, 290, 4000)])
def test_dgemm_vs_fp64_reference(api, opA, opB, M, N, K):
    rng = np.random.default_rng(M * 1000 + N * 10 + K)
    A = rng.standard_normal((M, K) if opA == 0 else (K, M))
    B = rng.standard_normal((K, N) if opB == 0 else (N, K))
    C0 = rng.standard_normal((M, N))
    ref = 1.5 * (A if opA == 0 else A.T) @ (B if opB == 0 else B.T) - 0.5 * C0
    C = _cm(C0)
    ws = torch.empty(1 << 22, dtype=torch.float64, device="cuda")
    api.dgemm(opA, opB, 1.5, _cm(A), _cm(B), -0.5, C, ws=ws)
    got = C.cpu().numpy()
    err = np.abs(got - ref).max() / (np.abs(A).max() * np.abs(B).max() * K + 1)
    assert err < 1e-15, err


def test_dgemm_odd_leading_dims(api):
    rng = np.random.default_rng(3)
    M, N, K = 37, 19, 51
    Abig = rng.standard_normal((M + 3, K))  # lda = 40 -> use an odd-ld view
    A = torch.from_numpy(np.ascontiguousarray(Abig.T)).cuda().T[:M, :]  # ld 40
    Bfull = torch.from_numpy(np.ascontiguousarray(rng.standard_normal((N, K + 1)))).cuda().T[:K, :]  # ld 52
    C = api.colmajor(M, N, ld=M)
    api.dgemm(0, 0, 1.0, A, Bfull, 0.0, C)
    ref = A.cpu().numpy() @ Bfull.cpu().numpy()
    assert np.abs(C.cpu().numpy() - ref).max() < 1e-12


@pytest.mark.parametrize("s", [1, 2, 3, 17, 64, 112, 113, 200, 301])
def test_jacobi_eig(api, s):
    rng = np.random.default_rng(s)
    M = rng.standard_normal((s, s))
    A = (M + M.T) / 2
    w, V, sweeps = api.jacobi(_cm(A))
    w = w.cpu().numpy()
    V = V.cpu().numpy()
    ref = np.linalg.eigvalsh(A)
    assert sweeps > 0
    assert np.abs(np.sort(w) - ref).max() < 1e-12 * max(1, np.abs(ref).max()) * max(1, s / 10)
    assert np.linalg.norm(V.T @ V - np.eye(s)) < 1e-12 * s
    assert np.linalg.norm(V @ np.diag(w) @ V.T - A) < 1e-12 * np.linalg.norm(A) * max(1, s / 10)


def test_philox_raw_bit_exact(api):
    cnt = 1000
    out = api.philox_raw(cnt, 7, 11, 13, 0x12345678, 0x9abcdef0).cpu().numpy().view(np.uint32)
    i = np.arange(cnt, dtype=np.uint32)
    ref = np.stack(philox4x32_10(i, 7, 11, 13, 0x12345678, 0x9abcdef0), axis=1).reshape(-1)
    assert np.array_equal(out, ref)


def test_philox_gauss_matches_oracle(api):
    n, q = 301, 7
    got = api.philox_gauss(n, q, seed=99, stream_id=5, ctx=2, tag=3).cpu().numpy()
    ref = gaussian_block(n, q, 99, 5, ctx=2, tag=3)
    assert np.abs(got - ref).max() < 1e-13


@pytest.mark.parametrize("s,m", [(1, 1), (2, 2), (3, 1), (17, 17), (64, 20), (65, 65), (100, 33), (129, 129),
                                 (160, 60), (161, 161), (193, 64), (256, 90), (257, 257), (300, 100), (385, 128),
                                 (449, 150), (500, 170), (512, 512), (513, 171), (640, 220), (641, 120), (800, 260),
                                 (1100, 300), (2000, 200)])
def test_eigh_tridiagonal(api, s, m):
    rng = np.random.default_rng(1000 + s)
    M = rng.standard_normal((s, s))
    A = (M + M.T) / 2
    w, V, npos = api.eigh(_cm(A), m)
    w = w.cpu().numpy()
    V = V.cpu().numpy()
    ref = np.linalg.eigvalsh(A)[::-1][:m]
    scale = max(1.0, np.abs(ref).max())
    assert np.abs(w - ref).max() <= 1e-12 * scale * max(1, s / 20)
    assert npos == int(np.sum(np.linalg.eigvalsh(A) > 0))
    assert np.linalg.norm(V.T @ V - np.eye(m)) <= 1e-11 * max(1, s / 20)
    R = A @ V - V * w
    assert np.linalg.norm(R, axis=0).max() <= 1e-11 * scale * max(1, s / 20)


def test_eigh_clustered_spectrum(api):
    """Planted spectrum with a tight near-zero cluster (the C3-R regime of the RR pencil)."""
    from workloads.generators import haar_q, planted
    rng = np.random.default_rng(5)
    s = 240
    lam = np.concatenate([10.0 ** rng.uniform(-3, 2, 40), -(10.0 ** rng.uniform(-3, 2, 180)),
                          rng.uniform(-1e-9, 1e-9, 20)])
    A = planted(haar_q(rng, s), lam)
    m = 80
    w, V, npos = api.eigh(_cm(A), m)
    w = w.cpu().numpy()
    V = V.cpu().numpy()
    ref = np.sort(lam)[::-1][:m]
    assert np.abs(w - ref).max() <= 1e-12 * 100 * 5
    assert np.linalg.norm(V.T @ V - np.eye(m)) <= 1e-10
    assert np.linalg.norm(A @ V - V * w, axis=0).max() <= 1e-10 * 100


@pytest.mark.parametrize("s", [12, 200])
def test_eigh_repeated_eigenvalues(api, s):
    """Exactly repeated eigenvalues: inverse iteration vectors of one eigenspace are not
    orthogonal; the Newton-Schulz / clustered-MGS fallback must still return an orthonormal,
    diagonalising basis."""
    from workloads.generators import haar_q, planted
    rng = np.random.default_rng(77 + s)
    k = s // 4
    lam = np.concatenate([np.full(k, 2.0), np.full(k, -1.0), np.full(k, 0.5), rng.uniform(-3, 3, s - 3 * k)])
    A = planted(haar_q(rng, s), lam)
    m = s // 2
    w, V, npos = api.eigh(_cm(A), m)
    w = w.cpu().numpy()
    V = V.cpu().numpy()
    ref = np.sort(lam)[::-1][:m]
    assert np.abs(w - ref).max() <= 1e-12 * 3 * max(1, s / 20)
    assert np.linalg.norm(V.T @ V - np.eye(m)) <= 1e-11 * max(1, s / 20)
    assert np.linalg.norm(A @ V - V * w, axis=0).max() <= 1e-11 * 3 * max(1, s / 20)


@pytest.mark.parametrize("t", [1, 5, 8, 9, 64, 150, 301, 520, 700, 1100])
def test_cholesky_cluster(api, t):
    """a6 Cholesky (cluster kernel for t <= ~580, one CTA above) vs LAPACK on an SPD Gram matrix."""
    rng = np.random.default_rng(300 + t)
    M = rng.standard_normal((t + 20, t))
    G = M.T @ M
    L, rc = api.cholesky(_cm(G))
    assert rc == 0
    L = L.cpu().numpy()
    ref = np.linalg.cholesky(G)
    assert np.abs(np.triu(L, 1)).max() == 0.0
    assert np.linalg.norm(L - ref) <= 1e-12 * np.linalg.norm(ref) * max(1, t / 10)


def test_cholesky_breakdown(api):
    """Rank-deficient Gram (two equal columns): the failing pivot is reported (R20)."""
    rng = np.random.default_rng(9)
    M = rng.standard_normal((40, 30))
    M[:, 17] = M[:, 3]
    L, rc = api.cholesky(_cm(M.T @ M))
    assert rc == 18


@pytest.mark.parametrize("s", [4, 40, 100])
@pytest.mark.parametrize("scale", [0.0, 1e-300, 1e300])
def test_eigh_extreme_scales(api, s, scale):
    """Sturm counts and eigenvalues at the ends of the exponent range (the bisection pre-scales T by
    a power of two; the zero matrix has no positive eigenvalue). Absolute accuracy floor: the
    bisection stops at a bracket of 4 pivmin ~ 1e-306 (dstebz's safe-minimum floor)."""
    A = np.diag(np.linspace(0.0, 1.0, s) * scale)
    w, V, npos = api.eigh(_cm(A), s)
    ref = np.sort(np.diag(A))[::-1]
    assert npos == int(np.sum(ref > 0))
    assert np.abs(w.cpu().numpy() - ref).max() <= 1e-13 * scale * s + 1e-306


@pytest.mark.parametrize("n,k", [(64, 1), (130, 7), (1000, 33), (1000, 64), (2048, 100), (4000, 70), (4000, 200),
                                 (998, 17), (4000, 17), (4000, 32), (4000, 56), (4002, 64), (3998, 45), (4096, 33), (4000, 9)])
@pytest.mark.parametrize("split", [False, True])
def test_symm_multiply_tma(api, n, k, split):
    """a3 block multiply on TMA-staged swizzled tiles (psdproj_symm_multiply, the kernel the path
    runs) against an fp64 reference: ragged m / k / column tiles come from the TMA zero fill. n >= 3520
    with 16 < k <= 64 takes the row-panel kernel (whole k range per CTA, in-CTA k-group sums)."""
    rng = np.random.default_rng(n + k)
    M = rng.standard_normal((n, n))
    A = (M + M.T) / 2
    Z = rng.standard_normal((n, k))
    Ad = torch.from_numpy(A).cuda()
    Zd = api.colmajor(n, k)
    Zd.copy_(torch.from_numpy(Z))
    ws = torch.empty(32 * n * k, dtype=torch.float64, device="cuda") if split else None
    Y = api.symm_multiply(-1.0, Ad, Zd, ws=ws).cpu().numpy()
    ref = -(A @ Z)
    assert np.abs(Y - ref).max() <= 1e-13 * np.sqrt(n) * np.abs(ref).max()


def test_eigh_two_stage_reduction_subprocess():
    """The optional two-stage tridiagonalisation (sbr.cuh, PSDPROJ_SBR=1: dense -> band on a cluster,
    band -> tridiagonal by bulge chasing, back-transformation through both) against LAPACK. The
    switch is read once per process, hence the subprocess (tools/sbr_probe.py)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PSDPROJ_SBR="1", PROBE_REPS="1")
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "sbr_probe.py"), "48,100,161,272,384"],
                         env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("s=")]
    assert len(lines) == 5, out.stdout
    for l in lines:
        f = dict(kv.split("=") for kv in l.split())
        s = int(f["s"])
        assert float(f["eig_relerr"]) <= 1e-13, l
        assert float(f["orth"]) <= 1e-12 * max(1, s / 20), l
        assert float(f["resid"]) <= 1e-11 * max(1, s / 20), l
        assert f["npos_ok"] == "True", l


@pytest.mark.parametrize("env", [{"PSDPROJ_TRI_WARP": "128"}, {"PSDPROJ_TRI_WARP": "0"}])
def test_eigh_alternative_tridiagonalisations_subprocess(env):
    """The non-default small-s tridiagonalisations against LAPACK eigenvalues: the one-CTA warp-cyclic
    kernel's 4 x 8 register variant (s <= 128, PSDPROJ_TRI_WARP=128) and the tiled one-CTA kernel
    (PSDPROJ_TRI_WARP=0). The switches are read once per process, hence the subprocess."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "eigh_probe.py"), "3:3,17:17,64:50,65:65,100:80,128:128"],
                         env=dict(os.environ, **env), capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    recs = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(recs) == 6, out.stdout
    for r in recs:
        assert r["max_err"] <= 1e-12 * max(1, r["s"] / 20) * 3.0 * r["s"] ** 0.5, r
