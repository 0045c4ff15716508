#!/usr/bin/env python
"""bench.py -- warm LOBPCG PSD-cone projections/s at n = 4000 (BASELINE.json metric).

A "step" is one warm projection psdproj_project of the next matrix of the C3-R sequence
(configs[2] with the spectrum-preserving drift, R30; n = 4000, 5% positive
log-uniform [1e-3, 1e2], eps_t = 1e-2/t, tol 1e-7), RUN TO CONVERGENCE (status OK; max_iter
4000 is a safety cap, never reached on this window): every timed projection is bound-verified
and its error against the closed form Pi*_t is reported (outside the timed region). The
sequence is generated on the GPU before timing (step 0 is the cold call, then W warm-up steps,
then K timed steps; every step reads a distinct 128 MB matrix, larger than the 126 MB L2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c3r|c4|c5] [--shard] [--n N] [--tol T] [--max-iter M]

--gpus N > 1 without torchrun: the script launches N ranks itself (torch.distributed.run on
127.0.0.1). The default line at N > 1: every rank projects its own independent C3-R sequence
(independent cone blocks, no collective; weak scaling), barrier + max-over-ranks device time.
--workload c4: the 512-block batch split across ranks by LPT; --shard: one matrix row-sharded
(NCCL inside the library). --impl reference times the oracle (oracle/, plain CPU, numpy + C
Jacobi) on a bounded sample on this box's host cores; rank 0 only.
"""
import argparse
import json
import os
import math
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FP64 = os.path.join(ROOT, "profiles", "peaks_fp64_r01.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "r02", "ncu_a3_r02.json")      # ncu --set full, one a3 launch
NCU_TRI = os.path.join(ROOT, "profiles", "r02", "ncu_tri_reg_r02.json")     # ncu --set full, one tridiag_reg launch


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3r", choices=["c3r", "c1", "c2", "c2cl", "c3", "c4", "c5", "bo"])
    ap.add_argument("--c4-blocks", type=int, default=512)
    ap.add_argument("--c4-no-tiny", action="store_true", help="C4: every block through its own context (no f4 routing)")
    ap.add_argument("--c4-direct-n", type=int, default=0,
                    help="C4: blocks with 112 < n <= this use the exact DIRECT path (side = 2) instead of LOBPCG")
    ap.add_argument("--shard", action="store_true",
                    help="row-shard the single matrix across the ranks (NCCL inside libpsdproj; strong scaling)")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--tol", type=float, default=None)
    ap.add_argument("--max-iter", type=int, default=4000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the phase / cold / sched companion lines")
    ap.add_argument("--admm-max-iter", type=int, default=5000)
    ap.add_argument("--c5-exact", action="store_true", help="C5: also solve with exact (DIRECT) projections")
    ap.add_argument("--adapt-every", type=int, default=0)
    ap.add_argument("--tol-ratio", type=float, default=0.0)
    ap.add_argument("--late-t0", type=int, default=100, help="first step of the late-sequence companion (0: off)")
    ap.add_argument("--krylov-depth", type=int, default=1, help="R57 block-Krylov depth (1 = Alg. 3)")
    ap.add_argument("--krylov-max-active", type=int, default=0, help="R63: R57 directions only while |J| <= this")
    ap.add_argument("--no-r63", action="store_true", help="skip the R63 block-Krylov companion line")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample-iters", type=int, default=4)
    return ap.parse_args()


def workload(args):
    from workloads import generators as G
    if args.workload == "c3r":
        cfg = G.C3R(args.n or 4000)
        name = f"C3-R n={cfg.n} (configs[2] spectrum, spectrum-preserving drift eps_t=1e-2/t), tol {cfg.tol:g}"
    elif args.workload == "c3":
        cfg = G.C3(args.n or 4000)
        name = f"C3 literal n={cfg.n} (configs[2] additive drift), tol {cfg.tol:g}"
    elif args.workload == "c1":
        cfg = G.C1(args.n or 200)
        name = f"C1 n={cfg.n} (configs[0]), tol {cfg.tol:g}"
    elif args.workload == "c2cl":
        cfg = G.C2CL(args.n or 1000)
        name = f"C2-cl n={cfg.n} (configs[1] clustered variant, R31), tol {cfg.tol:g}"
    else:
        cfg = G.C2(args.n or 1000)
        name = f"C2 n={cfg.n} (configs[1]), tol {cfg.tol:g}"
    tol = args.tol if args.tol is not None else cfg.tol
    return cfg, name, tol


def gen_matrices(cfg, count, device):
    import torch
    from workloads import generators as G
    mats = []
    if cfg.kind == "rotation":
        for t, A, Q, lam in G.rotation_sequence(cfg, steps=count, device=device):
            mats.append(A.contiguous())
    else:
        for t, A, _ in G.drift_sequence(cfg, steps=count):
            mats.append(torch.from_numpy(A).to(device))
    return mats


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return rank, world, local, dist
    torch.cuda.set_device(0)
    return 0, 1, 0, None


def barrier(dist):
    if dist is not None:
        dist.barrier()


def max_over_ranks(dist, v):
    import torch
    if dist is None:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(dist, v):
    import torch
    if dist is None:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


PHASES = ["a3_block_multiply", "w_p_projection", "gram_pencil", "cholesky_pencil", "rr_tridiagonal", "rotation",
          "residual_norms", "host_locking_assembly", "rr_bisection", "rr_inverse_iteration", "rr_back_transform",
          "rr_reorth_and_coeffs"]


# Algorithmic flops of one warm C3-R projection at n = 4000, tol 1e-7 (library counters, mean over
# the bench's timed window, profiles/bench_r02.log): the reference arm has no GPU run to read them from.
NOMINAL_FLOPS_PER_PROJECTION = 1.9e12


def _oracle_sample_flops(n, trace, m0):
    """Algorithmic flops of the oracle's sampled iterations by the library's own counting
    (SURVEY §8.d.2): block multiply 2 n^2 a, Grams 2 n s^2, rotations 8 n m s, RR 11.33 s^3."""
    f = 2.0 * n * n * m0  # the initial Rayleigh-Ritz block multiply
    for (s_, a, locked, npos) in trace:
        m = max(s_ - 2 * a, 1)
        f += 2.0 * n * n * a + 2.0 * n * s_ * s_ + 8.0 * n * m * s_ + (9 + 1 / 3 + 2) * s_ ** 3
    return f


def cpu_baseline(cfg, tol, args, gpu_flops_per_proj, gpu_iters=None):
    """The oracle as it stands (oracle/lobpcg.py) on a bounded sample of the same workload: one warm
    projection of step 1 started from the exact top block of step 0 (planted Q), capped at
    `cpu-sample-iters` LOBPCG iterations. Its flop rate (the library's algorithmic counting applied
    to the oracle's own iterations) is scaled to the algorithmic flops of a whole warm projection as
    the GPU ran it: the first iterations of a warm call have the widest basis (s ~ 3m), so scaling
    by iteration count would overstate the oracle's time."""
    import numpy as np
    from oracle import lobpcg as OL
    from workloads import generators as G
    n = cfg.n
    if cfg.kind == "rotation":
        seq = G.rotation_sequence(cfg, steps=2)
        _, A0, Q0, lam = next(seq)
        _, A1, Q1, _ = next(seq)
    else:
        seq = G.drift_sequence(cfg, steps=2)
        _, A0, (Q0, lam) = next(seq)
        _, A1, _ = next(seq)
    order = np.argsort(-lam)
    p = int(np.sum(lam > 0))
    X0 = Q0[:, order[: p + max(1, int(np.ceil(0.1 * p)))]]
    t0 = time.perf_counter()
    res = OL.lobpcg_pos(A1, X0, tol, max_iter=args.cpu_sample_iters, m_max=(n + 2) // 3 + 1)
    dt = time.perf_counter() - t0
    fl = _oracle_sample_flops(n, res.trace, X0.shape[1])
    rate = fl / dt
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        cores = max(int(i.get("num_threads", 1)) for i in info) if info else 1
    except Exception:
        cores = os.cpu_count()
    t_proj = gpu_flops_per_proj / rate
    return {"value": 1.0 / t_proj, "unit": "projections/s", "cores": cores, "kind": "oracle",
            "sample": (f"oracle LOBPCG (numpy BLAS + C Jacobi) warm projection of step 1 (n={n}) from the exact "
                       f"step-0 block, first {res.iters} iterations ({dt:.1f} s, {rate / 1e9:.1f} algorithmic "
                       f"GFLOP/s) scaled to the {gpu_flops_per_proj / 1e12:.2f} TFLOP of a whole warm projection"
                       + (f" ({gpu_iters:.0f} iterations) as measured on the GPU" if gpu_iters else
                          " (nominal, NOMINAL_FLOPS_PER_PROJECTION)"))}


def run_reference(args):
    """--impl reference: the oracle as it stands on this box's host cores, same config / metric /
    unit as our arm; each step a bounded sample (cpu_baseline), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from workloads import generators as G
    cfg = G.C3R(args.n or 4000)
    tol = args.tol if args.tol is not None else cfg.tol
    name = (f"C3-R n={cfg.n} (configs[2] spectrum, spectrum-preserving drift eps_t=1e-2/t, R30), tol {tol:g}, "
            f"run to convergence (max_iter {args.max_iter})")
    steps = []
    for k in range(args.warmup + args.steps):
        cb = cpu_baseline(cfg, tol, argparse.Namespace(cpu_sample_iters=2), NOMINAL_FLOPS_PER_PROJECTION)
        if k >= args.warmup:
            steps.append(cb)
    v = statistics.median([s["value"] for s in steps])
    line = {"impl": "reference", "metric": "PSD-cone projections/sec (warm LOBPCG) at n=4000",
            "value": v, "unit": "projections/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 / v, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": {"workload": name, "n": cfg.n, "tol": tol,
                                                          "max_iter": args.max_iter},
            "cpu_baseline": {"value": v, "unit": "projections/s", "cores": steps[-1]["cores"], "kind": "oracle",
                             "sample": steps[-1]["sample"]},
            "e2e": {"value": v, "unit": "projections/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_c4_bench(args, rank, world, local, dist):
    """BASELINE configs[3]: 512 independent blocks sharded across ranks by LPT (no data-path
    collective, weak-in-blocks-per-GPU is not fixed: the 512-block job is split, so scaling is
    strong); one step = one round of every block, warm-started from the previous round."""
    import torch
    from paper_1912_02767_b200.multigpu import run_c4
    from workloads.generators import C4
    cfg = C4(args.c4_blocks)
    dev = torch.device("cuda", local)
    clocks = Clocks(local)
    clocks.start()
    paths = {}
    ms, proj, iters, worst = run_c4(cfg, rank, world, dist, dev, rounds=max(args.steps, 1),
                                    warmup=max(args.warmup, 0), tiny=not args.c4_no_tiny, paths=paths,
                                    direct_n=args.c4_direct_n,
                                    params=dict(krylov_depth=args.krylov_depth,
                                                krylov_max_active=args.krylov_max_active))
    ck = clocks.stop()
    if rank == 0:
        # whole-round roofline: rank 0's algorithmic flops / bytes against the round time
        try:
            p64 = float(json.load(open(PEAKS_FP64))["dgemm_tflops_burst"])
            hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        except Exception:
            p64, hbm = 35.46, 6650.0
        fl, by = paths.get("alg_flops_bytes_per_round", [0.0, 0.0])
        t_roof = max(by / (hbm * 1e9), fl / (p64 * 1e12))
        step_roof = {"frac": t_roof / (ms / max(args.steps, 1) / 1e3), "t_roof_ms": t_roof * 1e3, "flops": fl, "bytes": by,
                     "definition": "rank 0's blocks: max(bytes/HBM, flops/P64) / round time (SURVEY §8.d.1; the "
                                   "library's per-call algorithmic counters, nominal 9 n^3 for the one-launch tiny blocks)"}
        line = {"metric": "PSD-cone projections/sec (warm LOBPCG), C4 batch of independent blocks",
                "value": proj / (ms / 1e3), "unit": "projections/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / max(args.steps, 1), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"C4 {cfg.count} blocks n in {{50,100,200,400}} (configs[3]), tol {cfg.tol:g}",
                           "parallelism": f"batch-sharded LPT x{world}", "l2": "per-round drift, no flush"},
                "iters_per_projection": {"mean": iters}, "worst_status": worst, "clocks": ck,
                "step_roofline": step_roof,
                "paths_rank0": paths, "direct_n": args.c4_direct_n, "krylov_depth": args.krylov_depth,
                "routing": ("n <= 112: one launch of the one-CTA warm LOBPCG (f4) for all of them, blocks whose smaller side "
                            "outgrows its 8 columns projected exactly in one CTA (R50); n > 112: one context each, "
                            "psdproj_project_batched") if not args.c4_no_tiny else "every block: one context, psdproj_project_batched"}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_c5_bench(args, rank, world, local, dist):
    """BASELINE configs[4] (f1): approximate ADMM (Alg. 1) on the MaxCut SDP of an Erdos-Renyi
    graph, n = 2000, p = 0.01, +-1 weights, to primal/dual residual 1e-4 (R33); one warm LOBPCG
    projection of the 2000 x 2000 block per ADMM iteration with tolerance 10/k^1.01.
    One step = one ADMM iteration; the whole solve is timed (device events around the loop)."""
    import torch
    from paper_1912_02767_b200.admm import MaxCutADMM
    from workloads.generators import maxcut_graph
    n = args.n or 2000
    L = maxcut_graph(n=n, p_edge=0.01, seed=501)
    from paper_1912_02767_b200 import api
    kprm = (api.default_params(seed=1912, krylov_depth=args.krylov_depth, krylov_max_active=args.krylov_max_active)
            if args.krylov_depth > 1 else None)
    solver = MaxCutADMM(L, device=f"cuda:{local}", adapt_every=args.adapt_every, tol_ratio=args.tol_ratio, params=kprm)
    for _ in range(max(args.warmup, 0)):
        solver.step()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    k0 = solver.k
    out = solver.solve(eps=1e-4, max_iter=args.admm_max_iter)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    its = solver.k - k0
    companion = None
    if args.tol_ratio == 0.0 and args.adapt_every == 0:
        # R59 companion: projection tolerance tied to the ADMM residual (the paper's schedule stays the cap)
        s2 = MaxCutADMM(L, device=f"cuda:{local}", tol_ratio=0.01)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(st)
        o2 = s2.solve(eps=1e-4, max_iter=args.admm_max_iter)
        f1.record(st)
        torch.cuda.synchronize()
        companion = {"definition": "R59: LOBPCG tol = min(10/k^1.01, 0.01 min(r_prim, r_dual))",
                     "solve_s": f0.elapsed_time(f1) / 1e3, "admm_iters": o2["iters"], "r_prim": o2["r_prim"],
                     "r_dual": o2["r_dual"], "objective": o2["objective"],
                     "lobpcg_iters_per_admm_iter": o2["lobpcg_iters"] / max(o2["iters"], 1)}
        s2.close()
    exact = None
    if args.c5_exact:
        # the paper's comparison (Table 1: ADMM with exact projections) on the same GPU:
        # every projection through the library's exact DIRECT path (side = 2, tridiagonal eigensolver of A)
        s3 = MaxCutADMM(L, device=f"cuda:{local}", params=api.default_params(seed=1912, side=2))
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(st)
        o3 = s3.solve(eps=1e-4, max_iter=args.admm_max_iter)
        g1.record(st)
        torch.cuda.synchronize()
        es = g0.elapsed_time(g1) / 1e3
        exact = {"definition": "same ADMM, every projection exact (side = PSDPROJ_SIDE_DIRECT)", "solve_s": es,
                 "admm_iters": o3["iters"], "ms_per_admm_iter": 1e3 * es / max(o3["iters"], 1),
                 "r_prim": o3["r_prim"], "r_dual": o3["r_dual"], "objective": o3["objective"],
                 "speedup_time_to_eps_approx_over_exact": es / (ms / 1e3),
                 "speedup_per_admm_iter": (es / max(o3["iters"], 1)) / (ms / 1e3 / max(its, 1))}
        s3.close()
    if rank == 0:
        infos = solver.infos
        line = {"metric": "MaxCut SDP approximate-ADMM iterations/sec (one warm LOBPCG projection each), n=2000",
                "value": its / (ms / 1e3), "unit": "ADMM iterations/s", "n_gpus": 1, "steps": its,
                "warmup": args.warmup, "ms_per_step": ms / max(its, 1), "higher_is_better": True,
                "scaling": "none", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"C5 MaxCut SDP, ER n={n}, p=0.01, +-1 weights (configs[4]), eps 1e-4",
                           "rho": solver.rho, "sigma": solver.sigma, "alpha": solver.alpha,
                           "rho_adaptation": f"residual balancing every {args.adapt_every} iterations (R58; 0 = fixed)",
                           "projection_tol": f"min(10/k^1.01, {args.tol_ratio} x min ADMM residual) (R59; 0 = the paper's schedule)",
                           "rho_history": solver.rho_history},
                "solve_s": ms / 1e3, "admm_iters": out["iters"], "r_prim": out["r_prim"], "r_dual": out["r_dual"],
                "objective": out["objective"],
                "lobpcg_iters_per_admm_iter": sum(i["iters"] for i in infos) / max(len(infos), 1),
                "sides": sorted(set(i["side"] for i in infos)), "cold_calls": sum(i["cold"] for i in infos),
                "time_to_1e-4_s": ms / 1e3 if out["r_prim"] <= 1e-4 and out["r_dual"] <= 1e-4 else None,
                "r59_companion": companion, "exact_projection_admm": exact}
        print(json.dumps(line), flush=True)
    solver.close()


def run_sharded_bench(args, rank, world, local, dist):
    """One C3-R matrix row-sharded over the ranks: rank r holds a contiguous row block
    of every input; per iteration the library all-gathers W and all-reduces the Gram partials.
    Strong scaling: the job (K warm projections of the sequence) is fixed as N grows."""
    import torch
    from paper_1912_02767_b200 import api
    cfg, name, tol = workload(args)
    dev = torch.device("cuda", local)
    W, K = max(args.warmup, 0), max(args.steps, 1)
    total = 1 + W + K
    r0, nr = api.row_blocks(cfg.n, world)[rank]
    mats = [api.colmajor_copy(A[r0:r0 + nr]) for A in gen_matrices(cfg, total, dev)]
    torch.cuda.synchronize()
    if rank == 0:
        uid = api.nccl_uid()
    obj = [uid if rank == 0 else None]
    if dist is not None:
        dist.broadcast_object_list(obj, src=0)
    prm = api.default_params(max_iter=args.max_iter, profile=1, seed=1912, ctx_id=0,
                             krylov_depth=args.krylov_depth, krylov_max_active=args.krylov_max_active)
    ctx = api.ShardedContext(cfg.n, r0, nr, obj[0], rank, world, params=prm, device=dev)
    out = api.colmajor(nr, cfg.n, device=dev)
    for k in range(1 + W):
        ctx.project(mats[k], tol, out=out)
    torch.cuda.synchronize()
    barrier(dist)
    clocks = Clocks(local)
    clocks.start()
    st = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    infos = []
    ev0.record(st)
    for k in range(1 + W, total):
        _, inf = ctx.project(mats[k], tol, out=out)
        infos.append(inf)
    ev1.record(st)
    torch.cuda.synchronize()
    barrier(dist)
    ck = clocks.stop()
    ms = max_over_ranks(dist, ev0.elapsed_time(ev1))
    if rank == 0:
        iters = [i["iters"] for i in infos]
        amul_ms = sum(i["amul_ms"] for i in infos)
        amul_flops = sum(i["amul_flops"] for i in infos)
        line = {"metric": "PSD-cone projections/sec (warm LOBPCG) at n=4000, row-sharded single matrix",
                "value": K / (ms / 1e3), "unit": "projections/s", "n_gpus": world, "steps": K, "warmup": W,
                "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": name, "n": cfg.n, "tol": tol, "max_iter": args.max_iter,
                           "parallelism": f"row-sharded x{world} (NCCL all-gather of W, all-reduce of Grams)",
                           "l2": "distinct 128 MB input matrix per step (> 126 MB L2), no flush"},
                "a3_local_tflops": amul_flops / max(amul_ms, 1e-9) / 1e9,
                "iters_per_projection": {"mean": statistics.mean(iters)}, "status": [i["status"] for i in infos],
                "gpu_launches": sum(i["launches"] for i in infos), "clocks": ck}
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


def run_sequence(args, rank, world, local, dist):
    """Companion lines for BASELINE configs[0], configs[1] (C2, C2-cl) and the literal configs[2] (C3):
    the whole warm sequence (cfg.steps matrices; step 0 cold, untimed) projected at the config
    tolerance, device-timed per call; status counts, iterations and bounds reported."""
    import torch
    from paper_1912_02767_b200 import api
    cfg, name, tol = workload(args)
    dev = torch.device("cuda", local)
    steps = 3 if args.workload == "c3" else cfg.steps  # C3 literal: the first steps only
    mats = gen_matrices(cfg, steps, dev)
    ctx = api.Context(cfg.n, params=api.default_params(max_iter=args.max_iter, seed=1912 + rank,
                                                       krylov_depth=args.krylov_depth,
                                                       krylov_max_active=args.krylov_max_active), device=dev)
    out = torch.empty_like(mats[0])
    st = torch.cuda.current_stream()
    infos, ms = [], []
    for k, A in enumerate(mats):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        _, inf = ctx.project(A, tol, out=out)
        e1.record(st)
        torch.cuda.synchronize()
        if k > 0:
            infos.append(inf)
            ms.append(e0.elapsed_time(e1))
    # the library's own exact path on the same matrices (side = PSDPROJ_SIDE_DIRECT, a13): where the
    # crossover between warm LOBPCG and the exact projection sits on this GPU (first 20 steps)
    direct = None
    if cfg.n <= 2000 and args.workload != "c3":
        dctx = api.Context(cfg.n, params=api.default_params(seed=1912 + rank, side=2), device=dev)
        dms, dinf = [], []
        for k, A in enumerate(mats[:21]):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _, inf = dctx.project(A, tol, out=out)
            e1.record(st)
            torch.cuda.synchronize()
            if k > 0:
                dms.append(e0.elapsed_time(e1))
                dinf.append(inf)
        dctx.close()
        direct = {"definition": "exact DIRECT path (a13) on steps 1..20 of the same sequence",
                  "value": len(dms) / (sum(dms) / 1e3), "unit": "projections/s", "ms_per_step": sum(dms) / len(dms),
                  "err_bound_rel_max": max(i["err_bound"] / i["anorm_f"] for i in dinf),
                  "status_counts": {str(s_): [i["status"] for i in dinf].count(s_)
                                    for s_ in sorted(set(i["status"] for i in dinf))}}
    if rank == 0:
        status = [i["status"] for i in infos]
        line = {"metric": f"PSD-cone projections/sec (warm LOBPCG), {name}", "value": len(ms) / (sum(ms) / 1e3),
                "unit": "projections/s", "n_gpus": 1, "steps": len(ms), "warmup": 0,
                "ms_per_step": sum(ms) / len(ms), "higher_is_better": True, "scaling": "none", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "config": {"workload": name, "n": cfg.n, "tol": tol},
                "iters_per_projection": {"mean": sum(i["iters"] for i in infos) / len(infos),
                                         "max": max(i["iters"] for i in infos)},
                "status_counts": {str(s_): status.count(s_) for s_ in sorted(set(status))},
                "err_bound_rel_max": max(i["err_bound"] / i["anorm_f"] for i in infos),
                "npos": sorted(set(i["npos"] for i in infos)), "sides": sorted(set(i["side"] for i in infos)),
                "exact_direct_companion": direct}
        print(json.dumps(line), flush=True)
    ctx.close()


def run_bo(args):
    """f4 line: BO-like tiny blocks (workloads.generators.BO), one-CTA warm LOBPCG per block vs the exact
    one-CTA Jacobi path, blocks/s per round (tools/tiny_lobpcg_probe.py)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "tiny_lobpcg_probe.py"), "4096", "8", "100",
                          str(max(args.steps, 3))], capture_output=True, text=True)
    print(out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-2000:], flush=True)


def spawn_ranks(args):
    """--gpus N without a torchrun environment: launch N ranks of this script with torchrun
    (one process per GPU, rendezvous on 127.0.0.1) and wait; rank 0 prints the JSON line."""
    import random
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={random.randint(20000, 40000)}", os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    return subprocess.call(cmd)


def accuracy(outs, mats, cfg):
    """Outside the timed region: rel_err = ||Pi~ - Pi*_t||_F / ||A_t||_F against the C3-R closed form
    Pi*_t = Q_t max(Lambda, 0) Q_t^T, on the GPU with torch."""
    import torch
    out = []
    for P, (A, Q, lam) in zip(outs, mats):
        Ps = (Q * torch.clamp(lam, min=0)) @ Q.T
        out.append(float(torch.linalg.norm(P - Ps)) / float(torch.linalg.norm(A)))
    return out


def run_c3r(args, rank, world, local, dist):
    import torch
    from paper_1912_02767_b200 import api
    from workloads import generators as G
    cfg = G.C3R(args.n or 4000)
    tol = args.tol if args.tol is not None else cfg.tol
    max_iter = args.max_iter
    name = (f"C3-R n={cfg.n} (configs[2] spectrum: 5% positive log-uniform [1e-3,1e2], negatives mirrored; "
            f"spectrum-preserving drift eps_t=1e-2/t, R30), tol {tol:g}, run to convergence (max_iter {max_iter})")
    dev = torch.device("cuda", local)
    W, K = max(args.warmup, 0), max(args.steps, 1)
    total = 1 + W + K
    # each rank projects its own independent sequence (weak scaling over independent cone blocks)
    cfg.seed = cfg.seed + 1000 * rank
    seq = []
    for t, A, Q, lam in G.rotation_sequence(cfg, steps=total, device=dev):
        seq.append((A.contiguous(), Q, lam))
    mats = [x[0] for x in seq]
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    kry = dict(krylov_depth=args.krylov_depth, krylov_max_active=args.krylov_max_active)
    prm = api.default_params(max_iter=max_iter, profile=5, seed=1912 + rank, ctx_id=rank, **kry)
    ctx = api.Context(cfg.n, params=prm, device=dev)
    outs = [torch.empty_like(mats[0]) for _ in range(K)]
    scratch = torch.empty_like(mats[0])
    infos_warm = []
    for k in range(1 + W):          # step 0 cold, then W warm-up steps (untimed)
        _, inf = ctx.project(mats[k], tol, out=scratch)
        infos_warm.append(inf)
    torch.cuda.synchronize()
    barrier(dist)
    clocks = Clocks(local)
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    evk = [torch.cuda.Event(enable_timing=True) for _ in range(K - 1)]
    infos = []
    torch.cuda.synchronize()
    barrier(dist)
    ev0.record(st)
    for j, k in enumerate(range(1 + W, total)):
        _, inf = ctx.project(mats[k], tol, out=outs[j])
        infos.append(inf)
        if j < K - 1:
            evk[j].record(st)
    ev1.record(st)
    torch.cuda.synchronize()
    barrier(dist)
    ck = clocks.stop()
    ms_local = ev0.elapsed_time(ev1)
    bounds = [ev0] + evk + [ev1]
    call_ms = sorted(bounds[j].elapsed_time(bounds[j + 1]) for j in range(K))
    ms = max_over_ranks(dist, ms_local)
    projections = sum_over_ranks(dist, float(K))
    value = projections / (ms / 1e3)
    rel = accuracy(outs, seq[1 + W:], cfg)
    del outs

    # dominant kernel: whichever of the a3 block multiply and the RR tridiagonalisation took more device
    # time (CUDA events on the launching stream around every launch, library profile bits 0 and 2)
    peaks = json.load(open(PEAKS_FP64))
    p64 = float(peaks["dgemm_tflops_burst"])
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm, hbm_src = float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        hbm, hbm_src = 6650.0, "fallback (B200_PROFILING.md)"
    amul_ms = sum(i["amul_ms"] for i in infos)
    amul_n = sum(i["amul_launches"] for i in infos)
    amul_flops = sum(i["amul_flops"] for i in infos)
    amul_bytes = sum(i["amul_bytes"] for i in infos)
    tri_ms = sum(i["tri_ms"] for i in infos)
    tri_n = sum(i["tri_launches"] for i in infos)
    tri_flops = sum(i["tri_flops"] for i in infos)
    cols = sum(i["a_cols"] for i in infos) / max(1, sum(i["a_passes"] for i in infos))
    def _load(path):
        try:
            return json.load(open(path))
        except Exception:
            return {}
    ncu, ncu_tri = _load(NCU_SUMMARY), _load(NCU_TRI)
    if tri_ms >= amul_ms:
        achieved = tri_flops / (tri_ms / 1e3) / 1e12 if tri_ms > 0 else 0.0
        roof = {"bound": "alu", "achieved": achieved, "peak": p64, "unit": "TFLOP/s", "frac": achieved / p64,
                "traffic": ncu_tri.get("dram_bytes_per_launch"),
                "traffic_source": "profiles/r02/ncu_tri_reg_r02.json (one launch, ncu --set full)",
                "kernel": "RR Householder tridiagonalisation (tridiag_reg_kernel: 16-CTA cluster, DSMEM pushes)",
                "share_of_step": tri_ms / ms_local,
                "per_launch": {"flops": tri_flops / max(1, tri_n), "ms": tri_ms / max(1, tri_n),
                               "launches": tri_n, "mean_s": (tri_flops / max(1, tri_n) * 0.75) ** (1 / 3)},
                "peak_source": "measured cuBLAS DGEMM 8192^3, FP64 (profiles/peaks_fp64_r01.json); the kernel is "
                               "latency-bound (one Householder column per dependent step), DESIGN.md §6"}
    else:
        achieved = amul_flops / (amul_ms / 1e3) / 1e12 if amul_ms > 0 else 0.0
        roof = {"bound": "tensor", "achieved": achieved, "peak": p64, "unit": "TFLOP/s", "frac": achieved / p64,
                "traffic": ncu.get("dram_bytes_per_launch"),
                "kernel": "a3 block multiply B.Z (dgemm_kp_kernel, DMMA)", "share_of_step": amul_ms / ms_local,
                "per_launch": {"mean_cols": cols, "flops": amul_flops / max(1, amul_n), "ms": amul_ms / max(1, amul_n)},
                "peak_source": "measured cuBLAS DGEMM 8192^3 (profiles/peaks_fp64_r01.json)"}
    a3 = {"achieved_tflops": amul_flops / (amul_ms / 1e3) / 1e12 if amul_ms > 0 else 0.0,
          "frac": (amul_flops / (amul_ms / 1e3) / 1e12 / p64) if amul_ms > 0 else 0.0,
          "share_of_step": amul_ms / ms_local, "mean_cols": cols, "launches": amul_n}
    flops = sum(i["flops"] for i in infos)
    byts = sum(i["bytes"] for i in infos)
    t_roof = max(byts / (hbm * 1e9), flops / (p64 * 1e12))
    iters = [i["iters"] for i in infos]
    status = [i["status"] for i in infos]
    bound_rel = [i["err_bound"] / i["anorm_f"] for i in infos]
    gpu_launches = sum(i["launches"] for i in infos)

    extra = {}
    if rank == 0 and not args.no_extra:
        extra = side_lines(args, cfg, tol, mats, seq, W, K, dev, api)

    e2e = None
    if not args.no_e2e:
        hprm = api.default_params(max_iter=max_iter, seed=1912 + rank, ctx_id=rank, host_io=1, **kry)
        hctx = api.Context(cfg.n, params=hprm, device=dev)
        ke_n = min(K, 3)
        host_mats = [m.cpu().pin_memory() for m in mats[: 1 + W + ke_n]]
        hout = torch.empty_like(host_mats[0]).pin_memory()
        for k in range(1 + W):
            hctx.project_host(host_mats[k], tol, out_host=hout)
        torch.cuda.synchronize()
        barrier(dist)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ke = 0
        for k in range(1 + W, len(host_mats)):
            hctx.project_host(host_mats[k], tol, out_host=hout)
            ke += 1
        e1.record(st)
        torch.cuda.synchronize()
        barrier(dist)
        ems = max_over_ranks(dist, e0.elapsed_time(e1))
        eproj = sum_over_ranks(dist, float(ke))
        nb = 8.0 * cfg.n * cfg.n
        e2e = {"value": eproj / (ems / 1e3), "unit": "projections/s", "h2d_bytes_per_step": nb,
               "d2h_bytes_per_step": nb, "steps": ke,
               "path": "psdproj_project_host (pinned host A and Pi, H2D + projection + D2H inside the call)"}
        hctx.close()

    if rank == 0:
        line = {
            "metric": "PSD-cone projections/sec (warm LOBPCG) at n=4000",
            "value": value, "unit": "projections/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "n": cfg.n, "tol": tol, "max_iter": max_iter, "locking": "hard",
                       "trial_space": ("Alg. 3 span(X, R, dX)" if args.krylov_depth <= 1 else
                                       f"R57/R63 span(X, R, .., B^{args.krylov_depth - 1} R, dX) while |J| <= "
                                       f"{args.krylov_max_active or 'inf'}, else Alg. 3"),
                       "steps_timed": f"t={1 + W}..{total - 1} of the sequence (t=0 cold, untimed)",
                       "parallelism": f"independent sequences x{world} (one per GPU, no collective)" if world > 1 else "single",
                       "l2": "distinct 128 MB input matrix per step (> 126 MB L2), no flush"},
            "accuracy": {"rel_err_vs_closed_form": rel, "max_rel_err": max(rel),
                         "err_bound_rel": bound_rel, "bound_dominates": all(b >= r for b, r in zip(bound_rel, rel)),
                         "npos": [i["npos"] for i in infos], "npos_true": int(round(0.05 * cfg.n)),
                         "status_counts": {str(s_): status.count(s_) for s_ in sorted(set(status))},
                         "oracle_matching_1e-9": max(rel) <= 1e-9},
            "roofline": roof,
            "a3_block_multiply": a3,
            "step_roofline": {"frac": t_roof / (ms_local / 1e3), "t_roof_ms": t_roof * 1e3 / K, "flops": flops / K,
                              "bytes": byts / K, "definition": "max(bytes/HBM, flops/P64) / step time (SURVEY §8.d.1)"},
            "per_call_ms": {"median": round(statistics.median(call_ms), 3),
                            "p90": round(call_ms[min(K - 1, int(math.ceil(0.9 * K)) - 1)], 3)},
            "iters_per_projection": {"warm_mean": statistics.mean(iters), "warm": iters,
                                     "cold_step0": infos_warm[0]["iters"]},
            "ms_per_iteration": ms / K / statistics.mean(iters),
            "gpu_launches": gpu_launches,
            "clocks": ck,
            "e2e": e2e,
            "profile_in_timed_region": "bits 0 and 2 only (2 CUDA events around each a3 and each tridiagonalisation launch)",
        }
        line.update(extra)
        if not args.no_cpu and world == 1:
            line["cpu_baseline"] = cpu_baseline(cfg, tol, args, flops / K, statistics.mean(iters))
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


def side_lines(args, cfg, tol, mats, seq, W, K, dev, api):
    """Untimed-for-the-headline companions, rank 0 only (each timed with its own CUDA events):
      phases     per-phase device time of the same warm steps (profile bit 1, a separate context
                 replaying the sequence: phase events stay out of the headline's timed region)
      cold       the first timed step's matrix projected cold (fresh context = after psdproj_reset)
      sched      C3-R-sched: the paper's tolerance schedule tol_t = 10 / t^1.01"""
    import torch
    out = {}
    st = torch.cuda.current_stream()
    kry = dict(krylov_depth=args.krylov_depth, krylov_max_active=args.krylov_max_active)
    prm = api.default_params(max_iter=args.max_iter, profile=2, seed=1912, ctx_id=0, **kry)
    pctx = api.Context(cfg.n, params=prm, device=dev)
    scratch = torch.empty_like(mats[0])
    infos = []
    for k in range(1 + W + K):
        _, inf = pctx.project(mats[k], tol, out=scratch)
        if k > W:
            infos.append(inf)
    ms = sum(sum(i["phase_ms"]) for i in infos) / len(infos)
    tot = {nm: round(sum(i["phase_ms"][j] for i in infos) / len(infos), 3) for j, nm in enumerate(PHASES)}
    out["phase_ms_per_step"] = tot
    dom = max(tot, key=tot.get)
    out["dominant_phase"] = {"phase": dom, "ms_per_step": tot[dom], "share": round(tot[dom] / max(ms, 1e-9), 4)}
    # late: the drift magnitudes of t = 100.. (eps_t = 1e-2/t) applied from the state of the last timed
    # step (Haar-invariant rotation: statistically the t = 100 state), warm from that step's block
    if args.late_t0 > 0:
        from workloads import generators as G
        lseq = [(A.contiguous(), Q, lam) for _, A, Q, lam in
                G.rotation_sequence(cfg, steps=4, device=dev, start=(seq[-1][1], seq[-1][2]), t0=args.late_t0 - 1)][1:]
        louts = [torch.empty_like(mats[0]) for _ in lseq]
        levs = [torch.cuda.Event(enable_timing=True) for _ in range(len(lseq) + 1)]
        linf = []
        torch.cuda.synchronize()
        levs[0].record(st)
        for j, (A, _, _) in enumerate(lseq):
            _, inf = pctx.project(A, tol, out=louts[j])
            linf.append(inf)
            levs[j + 1].record(st)
        torch.cuda.synchronize()
        lms = [levs[j].elapsed_time(levs[j + 1]) for j in range(len(lseq))]
        lrel = accuracy(louts, lseq, cfg)
        del louts
        out["late_sequence"] = {
            "definition": "drift eps_t = 1e-2/t of t = %d..%d applied after the last timed step (same tol, warm)"
                          % (args.late_t0, args.late_t0 + len(lseq) - 1),
            "value": len(lseq) / (sum(lms) / 1e3), "unit": "projections/s", "ms": [round(x, 3) for x in lms],
            "iters": [i["iters"] for i in linf], "status": [i["status"] for i in linf],
            "npos": [i["npos"] for i in linf], "rel_err_vs_closed_form": lrel,
            "err_bound_rel": [i["err_bound"] / i["anorm_f"] for i in linf]}
    # cold: same matrix as the first timed step, fresh context
    pctx.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    _, ci = pctx.project(mats[1 + W], tol, out=scratch)
    e1.record(st)
    torch.cuda.synchronize()
    out["cold_after_reset"] = {"t": 1 + W, "iters": ci["iters"], "ms": e0.elapsed_time(e1), "status": ci["status"],
                               "cold": ci["cold"]}
    pctx.close()
    # R63 companion: the same warm steps with block-Krylov directions while the active set is narrow
    # (krylov_depth 2, krylov_max_active 96; an extension of Alg. 3, off in the headline)
    if args.krylov_depth <= 1 and not args.no_r63:
        kprm = api.default_params(max_iter=args.max_iter, seed=1912, ctx_id=0, krylov_depth=2, krylov_max_active=96)
        kctx = api.Context(cfg.n, params=kprm, device=dev)
        kouts = [torch.empty_like(mats[0]) for _ in range(K)]
        kinf = []
        for k in range(1 + W):
            kctx.project(mats[k], tol, out=scratch)
        torch.cuda.synchronize()
        e0.record(st)
        for j, k in enumerate(range(1 + W, 1 + W + K)):
            _, inf = kctx.project(mats[k], tol, out=kouts[j])
            kinf.append(inf)
        e1.record(st)
        torch.cuda.synchronize()
        kms = e0.elapsed_time(e1)
        krel = accuracy(kouts, seq[1 + W:1 + W + K], cfg)
        del kouts
        kctx.close()
        out["r63_block_krylov"] = {
            "definition": "same timed steps, trial space span(X, R, B R, dX) on iterations with |J| <= 96 "
                          "(krylov_depth 2, krylov_max_active 96; DESIGN R57/R63), Alg. 3 otherwise",
            "value": K / (kms / 1e3), "unit": "projections/s", "ms_per_step": kms / K,
            "iters": [i["iters"] for i in kinf], "status": [i["status"] for i in kinf],
            "npos": [i["npos"] for i in kinf], "rel_err_vs_closed_form": krel,
            "err_bound_rel": [i["err_bound"] / i["anorm_f"] for i in kinf]}
    # timing context only (not a product path, no parity claim): the exact projection of
    # the first timed matrix by a library eigendecomposition on the same GPU (torch.linalg.eigh =
    # cuSOLVER syevd, then V+ Lambda+ V+^T) -- the GPU analogue of the paper's syevr baseline
    try:
        Ax = mats[1 + W]
        for rep in range(2):  # first pass warms cuSOLVER's workspace
            torch.cuda.synchronize()
            e0.record(st)
            lamx, Vx = torch.linalg.eigh(Ax)
            posx = lamx > 0
            Px = (Vx[:, posx] * lamx[posx]) @ Vx[:, posx].T
            e1.record(st)
            torch.cuda.synchronize()
        out["exact_eigh_context"] = {
            "definition": "torch.linalg.eigh (cuSOLVER) + V+ Lambda+ V+^T of the first timed matrix, same GPU; "
                          "library timing context, not the product path",
            "ms": e0.elapsed_time(e1), "npos": int(posx.sum())}
        del lamx, Vx, Px
    except Exception as ex:  # context line only: never fail the bench on it
        out["exact_eigh_context"] = {"unavailable": str(ex)[:200]}
    # C3-R-sched: tol_t = 10 / t^1.01 over the first steps of the same sequence (t >= 1)
    sprm = api.default_params(max_iter=args.max_iter, seed=1912, ctx_id=0, **kry)
    sctx = api.Context(cfg.n, params=sprm, device=dev)
    _, _ = sctx.project(mats[0], 10.0, out=scratch)
    souts = [torch.empty_like(mats[0]) for _ in range(1, len(mats))]
    rows = []
    e0.record(st)
    for k in range(1, len(mats)):
        _, inf = sctx.project(mats[k], 10.0 / k ** 1.01, out=souts[k - 1])
        rows.append((k, inf))
    e1.record(st)
    torch.cuda.synchronize()
    sms_ = e0.elapsed_time(e1)
    rel = accuracy(souts, seq[1:], cfg)
    del souts
    out["sched"] = {"definition": "C3-R-sched: tol_t = 10/t^1.01 (PAPER.md:507), same matrices t=1..%d" % (len(mats) - 1),
                    "value": len(rows) / (sms_ / 1e3), "unit": "projections/s",
                    "iters": [inf["iters"] for _, inf in rows], "status": [inf["status"] for _, inf in rows],
                    "npos": [inf["npos"] for _, inf in rows], "rel_err_vs_closed_form": rel,
                    "err_bound_rel": [inf["err_bound"] / inf["anorm_f"] for _, inf in rows],
                    "note": "the paper's bound ignores the perp term (PAPER.md:508): with the loose early tolerances "
                            "the block holds fewer than the 200 positives, so the reported bound need not dominate"}
    sctx.close()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
    import torch  # noqa: F401
    from paper_1912_02767_b200 import build as build_so
    build_so()  # no-op when libpsdproj.so is newer than its sources

    rank, world, local, dist = dist_setup(args)
    if args.workload == "c4":
        run_c4_bench(args, rank, world, local, dist)
        return
    if args.workload == "c5":
        run_c5_bench(args, rank, world, local, dist)
        return
    if args.shard:
        run_sharded_bench(args, rank, world, local, dist)
        return
    if args.workload == "bo":
        run_bo(args)
        return
    if args.workload in ("c1", "c2", "c2cl", "c3"):
        run_sequence(args, rank, world, local, dist)
        return
    run_c3r(args, rank, world, local, dist)


if __name__ == "__main__":
    main()
