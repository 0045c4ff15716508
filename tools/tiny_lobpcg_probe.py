"""f4 measurement: BO-like drifting blocks (workloads.generators.BO) projected per round by
(a) the one-CTA warm LOBPCG (psdproj_project_tiny_lobpcg) and (b) the exact one-CTA Jacobi path
(psdproj_project_tiny_batched); blocks/s of each (device time with CUDA events, rounds after warm-up).

  python tools/tiny_lobpcg_probe.py [count] [lo] [hi] [rounds]
"""
import json
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1912_02767_b200 import api  # noqa: E402
from workloads.generators import BO, planted  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 8
hi = int(sys.argv[3]) if len(sys.argv) > 3 else 100
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 5
cfg = BO(count, lo, hi)
mats = [torch.from_numpy(planted(*cfg.block(i))).cuda() for i in range(count)]
drifts = [[torch.from_numpy(cfg.drift(i, r)).cuda() for i in range(count)] for r in range(rounds + 2)]
outs = [torch.empty_like(a) for a in mats]
batch = api.TinyLobpcgBatch(cfg.sizes)
st = torch.cuda.current_stream()
res_l = {"ms": [], "iters": [], "status": []}
res_x = {"ms": []}
for r in range(rounds + 2):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(st)
    _, info = batch.project(mats, cfg.tol, outs=outs)
    e1.record(st)
    api.project_tiny_batched(mats, outs=outs)
    e2.record(st)
    torch.cuda.synchronize()
    if r >= 2:  # round 0 cold, round 1 first warm
        res_l["ms"].append(e0.elapsed_time(e1))
        res_l["iters"].append(float(np.mean(info["iters"])))
        res_l["status"].append({str(s): info["status"].count(s) for s in sorted(set(info["status"]))})
        res_x["ms"].append(e1.elapsed_time(e2))
    for i in range(count):
        mats[i] += drifts[r][i]
ml, mx = float(np.median(res_l["ms"])), float(np.median(res_x["ms"]))
print(json.dumps({"blocks": count, "n_range": [lo, hi], "rounds_timed": rounds,
                  "tiny_lobpcg": {"ms_per_round": ml, "blocks_per_s": count / (ml / 1e3), "mean_iters": res_l["iters"],
                                  "status": res_l["status"][-1]},
                  "exact_jacobi": {"ms_per_round": mx, "blocks_per_s": count / (mx / 1e3)},
                  "speedup": mx / ml}))
