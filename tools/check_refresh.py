import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1912_02767_b200 import api
rng = np.random.default_rng(3)
for n, npos in [(30, 4), (30, 8), (60, 10), (200, 20)]:
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.concatenate([rng.uniform(0.1, 2, npos), -rng.uniform(0.1, 2, n - npos)])
    lam[npos:npos + 3] = [-1e-6, -2e-6, -3e-6]  # near-zero negatives: long runs
    A = (Q * lam) @ Q.T
    At = torch.from_numpy(A).cuda()
    ctx = api.Context(n, params=api.default_params(seed=1, max_iter=200))
    ref = (Q * np.maximum(lam, 0)) @ Q.T
    for call in range(3):
        P, info = ctx.project(At, 1e-12)
        err = np.linalg.norm(P.cpu().numpy() - ref) / np.linalg.norm(ref)
        print(n, npos, call, "iters", info["iters"], "status", info["status"], "err", err, "bound", info["err_bound"], flush=True)
    ctx.close()
