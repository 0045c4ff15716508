"""C3-R convergence probe: per step iterations, status, time and the achieved error against the
closed form Pi*_t = Q_t max(Lambda, 0) Q_t^T, plus err_bound / ||A||_F.

  python tools/c3r_probe.py [--n 4000] [--steps 8] [--max-iter 4000] [--tol 1e-7] [--sched]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4000)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--max-iter", type=int, default=4000)
    ap.add_argument("--tol", type=float, default=1e-7)
    ap.add_argument("--sched", action="store_true", help="tol_t = 10 / t^1.01 (PAPER.md:507)")
    ap.add_argument("--reset-every", type=int, default=0)
    ap.add_argument("--param", action="append", default=[], help="name=value psdproj_params override")
    args = ap.parse_args()
    import torch
    from paper_1912_02767_b200 import api
    from workloads import generators as G
    cfg = G.C3R(args.n)
    kw = dict(max_iter=args.max_iter, profile=2, seed=1912)
    for p in args.param:
        k, v = p.split("=")
        kw[k] = float(v) if "." in v or "e" in v else int(v)
    prm = api.default_params(**kw)
    ctx = api.Context(cfg.n, params=prm)
    out = None
    for t, A, Q, lam in G.rotation_sequence(cfg, steps=args.steps, device="cuda"):
        tol = 10.0 / max(t, 1) ** 1.01 if args.sched else args.tol
        if args.reset_every and t % args.reset_every == 0:
            ctx.reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out, info = ctx.project(A, tol, out=out)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        Ps = (Q * torch.clamp(lam, min=0)) @ Q.T
        an = float(torch.linalg.norm(A))
        err = float(torch.linalg.norm(out - Ps))
        rec = {"t": t, "tol": tol, "status": info["status"], "iters": info["iters"], "cold": info["cold"],
               "ms": round(dt * 1e3, 1), "npos": info["npos"], "m": info["m"], "locked": info["locked"],
               "rr_max": info["rr_max"], "rel_err": err / an, "bound_rel": info["err_bound"] / an,
               "resid_max": info["resid_max"], "bound_ok": info["err_bound"] >= err,
               "phase_ms": [round(x, 1) for x in info["phase_ms"]]}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
