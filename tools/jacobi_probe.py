"""Time the path's Jacobi kernels (psdproj_jacobi) vs s; report sweeps and us/round."""
import os, sys, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1912_02767_b200 import api
for s in [int(x) for x in sys.argv[1].split(',')]:
    rng = np.random.default_rng(s)
    M = rng.standard_normal((s, s)); A = torch.from_numpy((M + M.T) / 2).cuda()
    w, V, sw = api.jacobi(A)  # warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); w, V, sw = api.jacobi(A); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    N = s + (s & 1)
    print(json.dumps({"s": s, "ctas": os.environ.get("PSDPROJ_JACOBI_CTAS", "all"), "ms": round(ms, 3), "sweeps": sw,
                      "us_per_round": round(1e3 * ms / max(1, sw * (N - 1)), 3)}), flush=True)
