#!/usr/bin/env python
"""bench.py -- warm LOBPCG PSD-cone projections/s at n = 4000 (BASELINE.json metric).

A "step" is one warm projection psdproj_project of the next matrix of the C3-R sequence
(configs[2] with the spectrum-preserving drift, R30; n = 4000, 5% positive
log-uniform [1e-3, 1e2], eps_t = 1e-2/t, tol 1e-7). The sequence is generated on the GPU
before timing (step 0 is the cold call, then W warm-up steps, then K timed steps; every step
reads a distinct 128 MB matrix, larger than the 126 MB L2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c3r|c1|c2|c3] [--n N] [--tol T] [--max-iter M]

N > 1 (torchrun): every rank runs its own replica of the sequence (the single-matrix path
does not shard yet) -- weak scaling, barrier + max-over-ranks device time.
--impl reference times the oracle (oracle/, plain CPU, numpy + C Jacobi) on a bounded sample
on this box's host cores; rank 0 only.
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
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_amul_r01.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3r", choices=["c3r", "c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--c4-blocks", type=int, default=512)
    ap.add_argument("--shard", action="store_true",
                    help="row-shard the single matrix across the ranks (NCCL inside libpsdproj; strong scaling)")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--tol", type=float, default=None)
    ap.add_argument("--max-iter", type=int, default=500)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample-iters", type=int, default=6)
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


def dominant_phase(infos, K, ms_step):
    """The phase that dominates a step (library profile bit 1, CUDA events on the launching stream).
    At n = 4000 it is the Rayleigh-Ritz tridiagonalisation: latency-bound (two one-way DSMEM
    pushes per Householder step), so its roof is the push-hop floor measured by
    tools/micro/push_bench2.cu (profiles/push_bench_r01.txt), not HBM or FP64."""
    tot = [sum(i["phase_ms"][k] for i in infos) / K for k in range(len(PHASES))]
    k = max(range(len(PHASES)), key=lambda j: tot[j])
    out = {"phase": PHASES[k], "ms_per_step": round(tot[k], 3), "share": round(tot[k] / ms_step, 4)}
    if PHASES[k] == "rr_tridiagonal":
        out.update({"bound": "latency", "kernel": "tridiag_reg_kernel (16-CTA cluster, matrix in registers, DSMEM bulk-copy + st.async pushes)",
                    "floor_note": "per Householder step >= 2 DSMEM hops (bulk-copy broadcast of v_j, st.async "
                                  "all-gather of p_j; ~0.9-1.2k cycles each, push_bench*) + the owner's Householder "
                                  "update and scalars = ~3k cycles; measured ~4.2k (s = 200) to ~5.5k (s = 400) "
                                  "cycles/step (PSDPROJ_TRI_PROF; profiles/ncu_r01/tridiag_reg_r01.json)"})
    return out


def cpu_baseline(cfg, tol, args, gpu_iters):
    """The oracle as it stands (oracle/lobpcg.py) on a bounded sample of the same workload:
    one warm projection of step 1 started from the exact top block of step 0 (planted Q),
    capped at `cpu-sample-iters` LOBPCG iterations; projections/s is scaled to the GPU's mean
    iterations per projection (the metric's unit)."""
    import numpy as np
    from oracle import lobpcg as OL
    from workloads import generators as G
    n = cfg.n
    if cfg.kind == "rotation":
        seq = G.rotation_sequence(cfg, steps=2)
        _, A0, Q0, lam = next(seq)
        _, A1, Q1, _ = next(seq)
        order = np.argsort(-lam)
        p = int(np.sum(lam > 0))
        X0 = Q0[:, order[: p + max(1, int(np.ceil(0.1 * p)))]]
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
    it = max(res.iters, 1)
    per_iter = dt / (it + 1)  # + the initial Rayleigh-Ritz pass
    iters_full = max(gpu_iters, 1.0)
    try:
        import threadpoolctl
        cores = max(int(i.get("num_threads", 1)) for i in threadpoolctl.threadpool_info()) if threadpoolctl.threadpool_info() else 1
    except Exception:
        cores = os.cpu_count()
    return {"value": 1.0 / (per_iter * (iters_full + 1)), "unit": "projections/s", "cores": cores,
            "kind": "oracle",
            "sample": (f"oracle LOBPCG warm projection of step 1 (n={n}) from the exact step-0 block, "
                       f"{it} iterations in {dt:.1f} s ({per_iter * 1e3:.0f} ms/iter), scaled to "
                       f"{iters_full:.0f} iterations/projection measured on the GPU")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg, name, tol = workload(args)
    # bounded sample per step: 3 iterations of the oracle's warm projection, scaled to max_iter
    steps = []
    for k in range(args.warmup + args.steps):
        cb = cpu_baseline(cfg, tol, argparse.Namespace(cpu_sample_iters=2), args.max_iter)
        if k >= args.warmup:
            steps.append(cb)
    v = statistics.median([s["value"] for s in steps])
    line = {"impl": "reference", "metric": "PSD-cone projections/sec (warm LOBPCG) at n=4000",
            "value": v, "unit": "projections/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 / v, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": {"workload": name, "n": cfg.n, "tol": tol,
                                                          "max_iter": args.max_iter},
            "cpu_baseline": {"value": v, "unit": "projections/s", "cores": steps[-1]["cores"], "kind": "oracle",
                             "sample": steps[-1]["sample"] + f"; reference arm assumes {args.max_iter} iterations"},
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
    ms, proj, iters, worst = run_c4(cfg, rank, world, dist, dev, rounds=max(args.steps, 1),
                                    warmup=max(args.warmup, 0))
    ck = clocks.stop()
    if rank == 0:
        line = {"metric": "PSD-cone projections/sec (warm LOBPCG), C4 batch of independent blocks",
                "value": proj / (ms / 1e3), "unit": "projections/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / max(args.steps, 1), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"C4 {cfg.count} blocks n in {{50,100,200,400}} (configs[3]), tol {cfg.tol:g}",
                           "parallelism": f"batch-sharded LPT x{world}", "l2": "per-round drift, no flush"},
                "iters_per_projection": {"mean": iters}, "worst_status": worst, "clocks": ck}
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
    solver = MaxCutADMM(L, device=f"cuda:{local}")
    for _ in range(max(args.warmup, 0)):
        solver.step()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    k0 = solver.k
    out = solver.solve(eps=1e-4, max_iter=args.max_iter if args.max_iter != 500 else 5000)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    its = solver.k - k0
    if rank == 0:
        infos = solver.infos
        line = {"metric": "MaxCut SDP approximate-ADMM iterations/sec (one warm LOBPCG projection each), n=2000",
                "value": its / (ms / 1e3), "unit": "ADMM iterations/s", "n_gpus": 1, "steps": its,
                "warmup": args.warmup, "ms_per_step": ms / max(its, 1), "higher_is_better": True,
                "scaling": "none", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"C5 MaxCut SDP, ER n={n}, p=0.01, +-1 weights (configs[4]), eps 1e-4",
                           "rho": solver.rho, "sigma": solver.sigma, "alpha": solver.alpha},
                "solve_s": ms / 1e3, "admm_iters": out["iters"], "r_prim": out["r_prim"], "r_dual": out["r_dual"],
                "objective": out["objective"],
                "lobpcg_iters_per_admm_iter": sum(i["iters"] for i in infos) / max(len(infos), 1),
                "sides": sorted(set(i["side"] for i in infos)), "cold_calls": sum(i["cold"] for i in infos)}
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
    prm = api.default_params(max_iter=args.max_iter, profile=1, seed=1912, ctx_id=0)
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


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    from paper_1912_02767_b200 import build as build_so
    build_so()  # no-op when libpsdproj.so is newer than its sources
    from paper_1912_02767_b200 import api

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
    cfg, name, tol = workload(args)
    dev = torch.device("cuda", local)
    W, K = max(args.warmup, 0), max(args.steps, 1)
    total = 1 + W + K
    mats = gen_matrices(cfg, total, dev)
    torch.cuda.synchronize()
    prm = api.default_params(max_iter=args.max_iter, profile=3, seed=1912 + rank, ctx_id=rank)
    ctx = api.Context(cfg.n, params=prm, device=dev)
    out = torch.empty_like(mats[0])
    st = torch.cuda.current_stream()
    # step 0: cold call; then W warm-up steps (untimed)
    infos_warm = []
    for k in range(1 + W):
        _, inf = ctx.project(mats[k], tol, out=out)
        infos_warm.append(inf)
    torch.cuda.synchronize()
    barrier(dist)
    clocks = Clocks(local)
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    infos = []
    torch.cuda.synchronize()
    barrier(dist)
    # per-call boundaries (events on the call's stream; no host sync inside the timed region)
    evk = [torch.cuda.Event(enable_timing=True) for _ in range(K - 1)]
    ev0.record(st)
    for j, k in enumerate(range(1 + W, total)):
        _, inf = ctx.project(mats[k], tol, out=out)
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

    # dominant kernel: the block multiply B.Z (a3)
    amul_ms = sum(i["amul_ms"] for i in infos)
    amul_launch = sum(i["amul_launches"] for i in infos)
    amul_flops = sum(i["amul_flops"] for i in infos)
    amul_bytes = sum(i["amul_bytes"] for i in infos)
    cols = sum(i["a_cols"] for i in infos) / max(1, sum(i["a_passes"] for i in infos))
    peaks = json.load(open(PEAKS_FP64))
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm = float(mp["hbm_gbs"])
        hbm_src = "measured (MEASURED_PEAKS.json)"
    except Exception:
        hbm = 6650.0
        hbm_src = "fallback (B200_PROFILING.md)"
    p64 = float(peaks["dgemm_tflops_burst"])
    intensity = 2.0 * cols / 8.0
    ridge = p64 * 1e12 / (hbm * 1e9)
    traffic = None
    if os.path.exists(NCU_SUMMARY):
        try:
            traffic = json.load(open(NCU_SUMMARY)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    if intensity >= ridge:
        achieved = amul_flops / (amul_ms / 1e3) / 1e12 if amul_ms > 0 else 0.0
        roof = {"bound": "tensor", "achieved": achieved, "peak": p64, "unit": "TFLOP/s",
                "frac": achieved / p64, "traffic": traffic,
                "kernel": "a3 block multiply B.Z (dgemm_kp_kernel, mma.sync m8n8k4 f64 = SASS DMMA.8x8x4 [+ split-K reduce])",
                "per_launch": {"mean_cols": cols, "flops": amul_flops / max(1, amul_launch),
                               "ms": amul_ms / max(1, amul_launch)},
                "peak_source": "measured cuBLAS DGEMM 8192^3 (profiles/peaks_fp64_r01.json)"}
    else:
        achieved = amul_bytes / (amul_ms / 1e3) / 1e9 if amul_ms > 0 else 0.0
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "kernel": "a3 block multiply B.Z",
                "per_launch": {"mean_cols": cols, "bytes": amul_bytes / max(1, amul_launch),
                               "ms": amul_ms / max(1, amul_launch)},
                "peak_source": hbm_src}
    # whole-step roofline (BASELINE metric: slower of bytes/HBM and flops/P64)
    flops = sum(i["flops"] for i in infos)
    byts = sum(i["bytes"] for i in infos)
    t_roof = max(byts / (hbm * 1e9), flops / (p64 * 1e12))
    step_frac = t_roof / (ms_local / 1e3)
    iters = [i["iters"] for i in infos]
    gpu_launches = sum(i["launches"] for i in infos)

    e2e = None
    if not args.no_e2e:
        hprm = api.default_params(max_iter=args.max_iter, seed=1912 + rank, ctx_id=rank, host_io=1)
        hctx = api.Context(cfg.n, params=hprm, device=dev)
        host_mats = [m.cpu().pin_memory() for m in mats[: 1 + W + min(K, 3)]]
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
               "d2h_bytes_per_step": nb, "steps": ke}
        hctx.close()

    if rank == 0:
        line = {
            "metric": "PSD-cone projections/sec (warm LOBPCG) at n=4000",
            "value": value, "unit": "projections/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "n": cfg.n, "tol": tol, "max_iter": args.max_iter,
                       "locking": "hard", "parallelism": f"replicas{world}" if world > 1 else "single",
                       "l2": "distinct 128 MB input matrix per step (> 126 MB L2), no flush"},
            "roofline": roof,
            "step_roofline": {"frac": step_frac, "t_roof_ms": t_roof * 1e3 / K, "flops": flops / K,
                              "bytes": byts / K, "definition": "max(bytes/HBM, flops/P64) / step time"},
            "per_call_ms": {"median": round(statistics.median(call_ms), 3),
                            "p90": round(call_ms[min(K - 1, int(math.ceil(0.9 * K)) - 1)], 3)},
            "phase_ms_per_step": {nm: round(sum(i["phase_ms"][k] for i in infos) / K, 3) for k, nm in enumerate(
                ["a3_block_multiply", "w_p_projection", "gram_pencil", "cholesky_pencil", "rr_tridiagonal",
                 "rotation", "residual_norms", "host_locking_assembly", "rr_bisection", "rr_inverse_iteration",
                 "rr_back_transform", "rr_reorth_and_coeffs"])},
            "dominant_phase": dominant_phase(infos, K, ms / K),
            "iters_per_projection": {"mean": statistics.mean(iters), "min": min(iters), "max": max(iters),
                                     "cold": infos_warm[0]["iters"]},
            "status": [i["status"] for i in infos],
            "gpu_launches": gpu_launches,
            "clocks": ck,
            "e2e": e2e,
        }
        if not args.no_cpu and world == 1:
            line["cpu_baseline"] = cpu_baseline(cfg, tol, args, statistics.mean(iters))
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
