import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1912_02767_b200 import api
from workloads.generators import haar_q, planted
rng = np.random.default_rng(22)
n, p = 300, 40
lam = np.concatenate([rng.uniform(0.5, 5, p), rng.uniform(-5, -0.5, n - p)])
Q = haar_q(rng, n)
A = planted(Q, lam)
Pstar = (Q * np.maximum(lam, 0)) @ Q.T
os.environ["PSDPROJ_TRACE"] = "1"
ctx = api.Context(n, params=api.default_params(seed=6, m0=8, expand_q=12, side=1))
Pi, info = ctx.project(torch.from_numpy(A).cuda(), 1e-10)
print({k: info[k] for k in ("status", "iters", "npos", "m", "expansions", "dropped", "locked", "err_bound")})
print("err", np.linalg.norm(Pi.cpu().numpy() - Pstar) / np.linalg.norm(A))
