"""Warm-sequence probe: per step iterations, status, time, positives for a BASELINE config.

  python tools/seq_probe.py --cfg c2cl --tol 1e-10 --steps 21 [--param keep_extra=20 ...] [--every 1]
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
    ap.add_argument("--cfg", default="c2")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--tol", type=float, default=None)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--every", type=int, default=1)
    ap.add_argument("--param", action="append", default=[])
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_1912_02767_b200 import api
    from workloads import generators as G
    kw = dict(max_iter=10000, seed=202)
    for p in args.param:
        k, v = p.split("=")
        kw[k] = float(v) if ("." in v or "e" in v) else int(v)
    mk = {"c1": G.C1, "c2": G.C2, "c2cl": G.C2CL, "c3r": G.C3R}[args.cfg]
    cfg = mk(args.n) if args.n else mk()
    tol = args.tol or cfg.tol
    ctx = api.Context(cfg.n, params=api.default_params(**kw))
    if cfg.kind == "rotation":
        it = ((t, A, (Q, lam)) for t, A, Q, lam in G.rotation_sequence(cfg, steps=args.steps, device="cuda"))
    else:
        it = ((t, torch.from_numpy(A).cuda(), x) for t, A, x in G.drift_sequence(cfg, steps=args.steps))
    for t, A, x in it:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, info = ctx.project(A, tol)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if t % args.every == 0:
            print(json.dumps({"t": t, "status": info["status"], "iters": info["iters"], "ms": round(1e3 * dt, 1),
                              "npos": info["npos"], "m": info["m"], "locked": info["locked"], "rr_max": info["rr_max"],
                              "bound_rel": info["err_bound"] / info["anorm_f"], "resid_max": info["resid_max"]}),
                  flush=True)


if __name__ == "__main__":
    main()
