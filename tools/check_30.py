import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1912_02767_b200 import api
rng = np.random.default_rng(3)
for n, npos in [(30, 4), (30, 8)]:
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.concatenate([rng.uniform(0.1, 2, npos), -rng.uniform(0.1, 2, n - npos)])
    lam[npos:npos + 3] = [-1e-6, -2e-6, -3e-6]
    A = (Q * lam) @ Q.T
    if npos != 8:
        continue
    np.save("gpurun_out/A30.npy", A)
    print("eigs", np.sort(lam)[::-1][:12])
    At = torch.from_numpy(A).cuda()
    os.environ["PSDPROJ_TRACE"] = "1"
    ctx = api.Context(n, params=api.default_params(seed=1, max_iter=60))
    P, info = ctx.project(At, 1e-12)
    print(info["iters"], info["status"], info["err_bound"])
