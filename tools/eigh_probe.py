"""Time the tridiagonal eigensolver (psdproj_eigh) vs s."""
import sys, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1912_02767_b200 import api
for spec in sys.argv[1].split(','):
    s, m = (int(x) for x in spec.split(':'))
    rng = np.random.default_rng(s)
    M = rng.standard_normal((s, s)); A = torch.from_numpy((M + M.T) / 2).cuda()
    api.eigh(A, m); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); w, V, npos = api.eigh(A, m); e1.record(); torch.cuda.synchronize()
    print(json.dumps({"s": s, "m": m, "ms": round(e0.elapsed_time(e1), 3)}), flush=True)
