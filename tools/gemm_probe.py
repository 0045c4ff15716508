"""Time the path's DMMA GEMM (psdproj_dgemm) on the shapes the LOBPCG iteration issues.
Usage: python tools/gemm_probe.py  (set PSDPROJ_GEMM=old for the first-cut kernel)"""
import json
import os
import sys

sys.path.insert(0, '.')
import torch

from paper_1912_02767_b200 import api

n = 4000
shapes = [("a3 NN", 0, 0, n, k, n) for k in (16, 32, 64, 87, 100, 128, 150, 200, 300)] + [
    ("gram TN", 1, 0, 400, 400, n), ("gram TN", 1, 0, 200, 200, n), ("rot NN", 0, 0, n, 200, 400),
    ("rot NN", 0, 0, n, 130, 330), ("orth NN", 0, 0, n, 110, 130), ("Pi NT", 0, 1, n, n, 200)]
ws = torch.empty(1 << 25, dtype=torch.float64, device="cuda")
for name, oa, ob, M, N, K in shapes:
    A = api.colmajor(K, M) if oa else api.colmajor(M, K)
    B = api.colmajor(N, K) if ob else api.colmajor(K, N)
    A.copy_(torch.randn(A.shape, dtype=torch.float64, device="cuda"))
    B.copy_(torch.randn(B.shape, dtype=torch.float64, device="cuda"))
    C = api.colmajor(M, N)
    opA = A.T if oa else A
    for _ in range(3):
        api.dgemm(oa, ob, 1.0, A, B, 0.0, C, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        api.dgemm(oa, ob, 1.0, A, B, 0.0, C, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ref = (A.T if oa else A) @ (B.T if ob else B)
    err = float((C - ref).abs().max() / ref.abs().max())
    print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "ms": round(ms, 4), "TF": round(2 * M * N * K / ms / 1e9, 2),
                      "relerr": err, "kernel": os.environ.get("PSDPROJ_GEMM", "kp")}), flush=True)
