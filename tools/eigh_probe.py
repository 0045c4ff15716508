"""Time the Rayleigh-Ritz eigensolver (psdproj_eigh, device time with CUDA events, min of 5) vs s.

  python tools/eigh_probe.py 64:20,128:40,...   (PSDPROJ_TRI_TILE=0 selects the cluster kernel)
"""
import json
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1912_02767_b200 import api  # noqa: E402

for spec in sys.argv[1].split(','):
    s, m = (int(x) for x in spec.split(':'))
    rng = np.random.default_rng(s)
    M = rng.standard_normal((s, s))
    A = torch.from_numpy((M + M.T) / 2).cuda()
    api.eigh(A, m)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        w, V, npos = api.eigh(A, m)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    ref = np.linalg.eigvalsh((M + M.T) / 2)[::-1][:m]
    err = float(np.abs(w.cpu().numpy() - ref).max())
    print(json.dumps({"s": s, "m": m, "ms": round(best, 3), "max_err": err}), flush=True)
