import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1912_02767_b200 import api
os.environ["PSDPROJ_TRACE"] = "1"
A = torch.zeros(40, 40, dtype=torch.float64, device="cuda")
ctx = api.Context(40, seed=1)
for call in range(3):
    try:
        P, info = ctx.project(A, 1e-10)
        print(call, {k: info[k] for k in ("status", "iters", "npos", "m", "dropped", "cold")}, flush=True)
    except Exception as ex:
        print(call, "ERR", ex, flush=True)
