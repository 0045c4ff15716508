"""Subprocess body of tests/test_sharded_loopback.py (TEST INFRASTRUCTURE): `world` ranks of the
row-sharded mode (psdproj_create_sharded) as host threads of ONE process on ONE GPU, collectives
through the in-process loopback NCCL (tests/nccl_loopback.cu, loaded via PSDPROJ_NCCL_LIB). Prints
one JSON line: per-step errors against O-EXACT and the unsharded context, cross-rank agreement."""
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.exact import project_exact  # noqa: E402
from paper_1912_02767_b200 import api  # noqa: E402
from workloads.generators import C1, drift_sequence, haar_q, planted  # noqa: E402


def main():
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    case = sys.argv[2] if len(sys.argv) > 2 else "c1"
    if case == "c1":
        cfg = C1()
        n, tol = cfg.n, 1e-10
        mats = [A for _, A, _ in drift_sequence(cfg, steps=4)]
    else:  # odd order, more positives, negative side
        rng = np.random.default_rng(5)
        n, tol = 333, 1e-10
        lam = np.concatenate([rng.uniform(0.1, 3, 300), rng.uniform(-3, -0.1, 33)])
        A0 = planted(haar_q(rng, n), lam)
        mats = [A0 + 1e-3 * k * np.eye(n) for k in range(3)]
    side = -1 if case != "c1" else 0
    uid = api.nccl_uid()
    blocks = api.row_blocks(n, world)
    results = [None] * world
    errors = [None] * world

    def run(rank):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                r0, nr = blocks[rank]
                ctx = api.ShardedContext(n, r0, nr, uid, rank, world, params=api.default_params(seed=13, side=side))
                outs = []
                for A in mats:
                    Ad = torch.from_numpy(A).cuda()
                    P, info = ctx.project(api.colmajor_copy(Ad[r0:r0 + nr]), tol)
                    torch.cuda.current_stream().synchronize()
                    outs.append((P.cpu().numpy(), info))
                ctx.close()
            results[rank] = outs
        except Exception as e:  # reported, not swallowed
            errors[rank] = repr(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if any(errors):
        print(json.dumps({"error": errors}))
        return
    un = api.Context(n, params=api.default_params(seed=13, side=side))
    rows = []
    for k, A in enumerate(mats):
        P = np.vstack([results[r][k][0] for r in range(world)])
        infos = [results[r][k][1] for r in range(world)]
        Pu, iu = un.project(torch.from_numpy(A).cuda(), tol)
        Pe = project_exact(A)
        nA = float(np.linalg.norm(A))
        keys = ("iters", "npos", "side", "status", "err_bound", "m", "locked")
        rows.append({
            "step": k,
            "rel_err_oracle": float(np.linalg.norm(P - Pe)) / nA,
            "rel_diff_unsharded": float(np.linalg.norm(P - Pu.cpu().numpy())) / nA,
            "err": float(np.linalg.norm(P - Pe)),
            "err_bound": infos[0]["err_bound"],
            "symmetric": bool(np.array_equal(P, P.T)),
            "ranks_agree": all(all(infos[r][kk] == infos[0][kk] for kk in keys) for r in range(world)),
            "iters": infos[0]["iters"], "iters_unsharded": iu["iters"], "npos": infos[0]["npos"],
            "side": infos[0]["side"], "status": infos[0]["status"],
        })
    un.close()
    print(json.dumps({"world": world, "n": n, "rows": rows}))


if __name__ == "__main__":
    main()
