"""Per-call LOBPCG statistics on a few C4 blocks over rounds (iterations, cold flag, side, drops)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1912_02767_b200 import api
from workloads.generators import C4, planted
cfg = C4(24)
for i in range(8):
    Q, lam = cfg.block(i)
    A = planted(Q, lam)
    ctx = api.Context(cfg.sizes[i], params=api.default_params(seed=1912, ctx_id=i))
    rows = []
    for r in range(4):
        _, info = ctx.project(torch.from_numpy(A).cuda(), cfg.tol)
        rows.append((info["iters"], info["cold"], info["side"], info["status"], info["dropped"], info["m"], info["expansions"]))
        A = A + cfg.drift(i, r)
    print(i, cfg.sizes[i], cfg.npos[i], rows, flush=True)
    ctx.close()
