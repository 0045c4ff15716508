"""One small call per path for compute-sanitizer runs (tools/sanitize.sh): eigh at s (cluster
tridiagonalisation for s > 64, tile kernel below), or a 3-step C1 projection sequence."""
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1912_02767_b200 import api  # noqa: E402

what = sys.argv[1]
if what == "eigh":
    s, m = int(sys.argv[2]), int(sys.argv[3])
    rng = np.random.default_rng(s)
    M = rng.standard_normal((s, s))
    w, V, npos = api.eigh(torch.from_numpy((M + M.T) / 2).cuda(), m)
    torch.cuda.synchronize()
    print("eigh", s, m, float(w[0]), npos)
elif what == "c1":
    from workloads.generators import C1, drift_sequence
    cfg = C1()
    ctx = api.Context(cfg.n, seed=11)
    for t, A, _ in drift_sequence(cfg, steps=3):
        _, info = ctx.project(torch.from_numpy(A).cuda(), 1e-10)
        print("c1", t, info["status"], info["iters"], info["err_bound"])
    ctx.close()
elif what == "chol":
    t = int(sys.argv[2])
    rng = np.random.default_rng(t)
    M = rng.standard_normal((t + 20, t))
    L, rc = api.cholesky(torch.from_numpy(M.T @ M).cuda())
    torch.cuda.synchronize()
    print("chol", t, rc)
