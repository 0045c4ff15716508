"""Trace the n=200 MaxCut ADMM (tests/test_admm.py) iteration by iteration: residuals and projection info."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1912_02767_b200.admm import MaxCutADMM
from paper_1912_02767_b200 import api
from workloads.generators import maxcut_graph
L = maxcut_graph(n=200, p_edge=0.05, seed=501)
solver = MaxCutADMM(L)
import os
tk = int(os.environ.get("TRACE_K", "-1"))
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 60):
    V_in = solver.V.clone()
    if k == tk:
        os.environ["PSDPROJ_TRACE"] = "1"
    rp, rd, info = solver.step()
    if k < 40 or k % 50 == 0:
        print(k, f"rp={rp:.3e} rd={rd:.3e}", {kk: info[kk] for kk in ("status", "iters", "npos", "m", "rr_max", "dropped", "err_bound", "resid_max", "lock_defect", "anorm_f", "locked", "expansions") if kk in info}, flush=True)
    if k == 5:
        Vin = V_in.cpu().numpy()
        Z = solver.Zp.cpu().numpy()
        w, Q = np.linalg.eigh(0.5 * (Vin + Vin.T))
        ref = (Q * np.maximum(w, 0)) @ Q.T
        print("proj err k=5", np.linalg.norm(Z - ref) / np.linalg.norm(ref), "npos", int((w > 0).sum()), flush=True)
