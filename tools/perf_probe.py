"""Per-call timing probe of the GPU path on C3-R-like sequences (development tool)."""
import sys, time, json
sys.path.insert(0, '.')
import torch
from paper_1912_02767_b200 import api
from workloads import generators as G
n = int(sys.argv[1]); steps = int(sys.argv[2]); mi = int(sys.argv[3]); tol = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-7
cfg = G.C3R(n)
mats = [A for _, A, _, _ in G.rotation_sequence(cfg, steps=steps, device='cuda')]
ctx = api.Context(n, params=api.default_params(max_iter=mi, profile=3))
out = torch.empty_like(mats[0])
for k, A in enumerate(mats):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _, inf = ctx.project(A, tol, out=out)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(json.dumps({"n": n, "k": k, "ms": round(dt*1e3, 2), "iters": inf["iters"], "status": inf["status"], "npos": inf["npos"],
          "rr_max": inf["rr_max"], "a_cols/it": round(inf["a_cols"]/max(1,inf["iters"]),1), "amul_ms": round(inf["amul_ms"],2),
          "amul_TF": round(inf["amul_flops"]/max(inf["amul_ms"],1e-9)/1e9, 2), "locked": inf["locked"], "launches": inf["launches"],
          "bound": inf["err_bound"], "m": inf["m"], "dropped": inf["dropped"], "phase_ms": [round(x, 2) for x in inf["phase_ms"]]}), flush=True)
