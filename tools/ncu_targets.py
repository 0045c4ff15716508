"""Small driver for ncu captures: one Jacobi (smem, s=64), one Jacobi (coop, s=300),
one a3 block multiply at n=4000, k=128 (DMMA GEMM)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1912_02767_b200 import api
what = sys.argv[1]
if what in ("jac64", "jac300"):
    s = 64 if what == "jac64" else 300
    rng = np.random.default_rng(s)
    M = rng.standard_normal((s, s)); A = torch.from_numpy((M + M.T) / 2).cuda()
    for _ in range(2):
        api.jacobi(A)
elif what == "amul":
    n, k = 4000, int(sys.argv[2]) if len(sys.argv) > 2 else 128
    A = torch.randn(n, n, dtype=torch.float64, device="cuda"); A = A + A.T
    Z = api.colmajor(n, k); Z.copy_(torch.randn(n, k, dtype=torch.float64, device="cuda"))
    Y = api.colmajor(n, k)
    ws = torch.empty(1 << 24, dtype=torch.float64, device="cuda")
    for _ in range(3):
        api.dgemm(0, 0, 1.0, A.T, Z, 0.0, Y, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        api.dgemm(0, 0, 1.0, A.T, Z, 0.0, Y, ws=ws)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"amul n={n} k={k}: {ms:.3f} ms, {2*n*n*k/ms/1e9:.2f} TF/s, {8*n*n/ms/1e6:.0f} GB/s")
torch.cuda.synchronize()
