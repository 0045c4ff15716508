"""Two-stage tridiagonalisation (sbr.cuh) probe: eigh accuracy vs LAPACK and eigensolver time per s.
Run twice, with PSDPROJ_SBR=1 and PSDPROJ_SBR=0, to compare against the one-stage cluster kernel."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_02767_b200 import api

sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "48,96,100,128,129,161,200,256,272,300,350,384").split(",")]
REPS = int(os.environ.get("PROBE_REPS", "20"))
for s in sizes:
    rng = np.random.default_rng(s)
    M = rng.standard_normal((s, s))
    A = (M + M.T) / 2
    At = torch.from_numpy(np.asfortranarray(A)).cuda()
    m = max(1, s // 3)
    w, V, npos = api.eigh(At, m)
    torch.cuda.synchronize()
    ref = np.linalg.eigvalsh(A)[::-1][:m]
    wv = w.cpu().numpy()
    Vn = V.cpu().numpy()
    ew = np.abs(wv - ref).max() / np.abs(ref).max()
    orth = np.linalg.norm(Vn.T @ Vn - np.eye(m))
    res = np.linalg.norm(A @ Vn - Vn * wv, axis=0).max()
    # timing: 20 calls
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(min(3, REPS)):
        api.eigh(At, m)
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(REPS):
        api.eigh(At, m)
    ev1.record()
    torch.cuda.synchronize()
    print(f"s={s} m={m} eig_relerr={ew:.2e} orth={orth:.2e} resid={res:.2e} npos_ok={npos == int((np.linalg.eigvalsh(A) > 0).sum())} "
          f"ms_per_eigh={ev0.elapsed_time(ev1) / REPS:.3f}", flush=True)
