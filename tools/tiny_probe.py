"""f4 throughput: many tiny blocks (n uniform in [lo, hi]) projected in one launch."""
import sys, json, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1912_02767_b200 import api
count, lo, hi = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(5)
mats = []
for n in rng.integers(lo, hi + 1, count):
    M = rng.standard_normal((n, n))
    mats.append(torch.from_numpy(0.5 * (M + M.T)).cuda())
outs = [torch.empty_like(a) for a in mats]
api.project_tiny_batched(mats, outs=outs)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    api.project_tiny_batched(mats, outs=outs)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(json.dumps({"blocks": count, "n_range": [lo, hi], "ms": round(min(ts) * 1e3, 3),
                  "blocks_per_s": round(count / min(ts), 1)}))
