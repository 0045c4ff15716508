"""f1 variants on the reduced C5 recipe (n = 200, p = 0.05) and the full C5 (n = 2000): iterations and
residuals for fixed rho / R58 / R59 combinations."""
import json
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_1912_02767_b200.admm import MaxCutADMM  # noqa: E402
from workloads.generators import maxcut_graph  # noqa: E402

n = int(sys.argv[1])
p = 0.05 if n <= 500 else 0.01
L = maxcut_graph(n=n, p_edge=p, seed=501)
for adapt, ratio in ((0, 0.0), (0, 0.01), (40, 0.01), (0, 0.1)):
    s = MaxCutADMM(L, adapt_every=adapt, tol_ratio=ratio)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = s.solve(eps=1e-4, max_iter=6000)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"n": n, "adapt_every": adapt, "tol_ratio": ratio, "iters": out["iters"], "s": round(dt, 2),
                      "r_prim": out["r_prim"], "r_dual": out["r_dual"], "objective": out["objective"],
                      "lobpcg_iters": out["lobpcg_iters"], "not_conv": sum(i["status"] == 1 for i in s.infos)}),
          flush=True)
    s.close()
