"""Batch sharding of independent cone blocks across GPUs (BASELINE configs[3]).

The paper projects every PSD block of a block-split SDP independently;
a batch of independent blocks shards with no data-path collective: each rank owns a fixed subset
of blocks (and their warm-start contexts) for every ADMM round, and only per-round scalars
(device time, iteration counts, worst status) cross ranks. One process per GPU; the process
group is torch.distributed (NCCL on the box, gloo in the CPU tests) and is used only for those
scalars and for the final gather of statistics.

Host logic only: the projections themselves run through api.project_batched (libpsdproj.so).
"""
import heapq
import time

import numpy as np


def block_cost(n, npos):
    """Relative cost of one warm projection of an n x n block with npos positive eigenvalues:
    LOBPCG on the smaller side costs ~ n^2 (p + guard) per iteration; a block with
    min(p, n - p) >= n/3 takes the DIRECT eigensolver path (~ n^3)."""
    p = min(npos, n - npos)
    if 3 * p >= n:
        return float(n) ** 3 / 8.0
    return float(n) ** 2 * (p + 16)


def lpt_partition(costs, world):
    """Longest-processing-time-first assignment of blocks to ranks. Deterministic: blocks in
    order of decreasing cost (ties by index), each to the least-loaded rank (ties by rank).
    Returns (list of block-index lists per rank, per-rank load)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    parts = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        parts[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    loads = [0.0] * world
    for r, p in enumerate(parts):
        loads[r] = sum(costs[i] for i in p)
        p.sort()
    return parts, loads


def lpt_bound(costs, world):
    """Graham's bound for LPT: makespan <= (4/3 - 1/(3 world)) OPT, OPT >= max(mean, max cost)."""
    opt_lb = max(sum(costs) / world, max(costs) if costs else 0.0)
    return (4.0 / 3.0 - 1.0 / (3.0 * world)) * opt_lb


TINY_NMAX = 112  # blocks up to this order go through the one-CTA path (tiny_lobpcg.cuh, TL_NMAX)


class C4Shard:
    """The blocks of BASELINE configs[3] (C4) owned by one rank: device matrices, the warm state
    across rounds, and the round-to-round drift. Blocks with n <= TINY_NMAX (tiny=True, default) are
    projected together by ONE launch of the one-CTA warm LOBPCG (psdproj_project_tiny_lobpcg, f4),
    which hands the blocks whose smaller side outgrows its 8-column block to the exact one-CTA
    projection (the DIRECT branch; R50); the others run one psdproj context each
    through psdproj_project_batched. direct_n > 0 (a routing option, off by default): the contexts of
    blocks with n <= direct_n are created with side = PSDPROJ_SIDE_DIRECT, i.e. the library's exact
    one-sided projection (a13) instead of LOBPCG -- at these sizes a round of the batch is bound by
    kernel launches (~50 per LOBPCG iteration), not by arithmetic (C4)."""

    def __init__(self, cfg, block_ids, device, seed=1912, max_iter=500, tiny=True, direct_n=0, params=None):
        import torch

        from . import api
        from workloads.generators import planted

        self.cfg = cfg
        self.ids = list(block_ids)
        self.device = device
        self.mats, self.outs = [], []
        for i in self.ids:
            Q, lam = cfg.block(i)
            A = torch.from_numpy(planted(Q, lam)).to(device)
            self.mats.append(A)
            self.outs.append(torch.empty_like(A))
        self.small = [k for k, i in enumerate(self.ids) if tiny and cfg.sizes[i] <= TINY_NMAX]
        self.large = [k for k in range(len(self.ids)) if k not in set(self.small)]
        self.ctxs = []
        for k in self.large:
            i = self.ids[k]
            prm = api.default_params(max_iter=max_iter, seed=seed, ctx_id=i,
                                     side=2 if cfg.sizes[i] <= direct_n else 0, **(params or {}))
            self.ctxs.append(api.Context(cfg.sizes[i], params=prm, device=device))
        self.tiny = (api.TinyLobpcgBatch([cfg.sizes[self.ids[k]] for k in self.small], device=device, seed=seed,
                                         max_iter=max_iter) if self.small else None)
        self.round = 0

    def drift(self):
        """A_{r+1} = A_r + 1e-3 sym(G) per block (R32); inputs generated outside timed regions."""
        import torch

        for k, i in enumerate(self.ids):
            self.mats[k] += torch.from_numpy(self.cfg.drift(i, self.round)).to(self.device)
        self.round += 1

    def project(self, tol=None):
        """One round: every block projected; per-block info dicts (iters, status, err_bound, path)."""
        from . import api

        tol = self.cfg.tol if tol is None else tol
        infos = [None] * len(self.ids)
        t0 = time.perf_counter()
        if self.small:
            _, res = self.tiny.project([self.mats[k] for k in self.small], tol,
                                       outs=[self.outs[k] for k in self.small])
            for j, k in enumerate(self.small):
                st = res["status"][j]
                # algorithmic work of a tiny block (counted here because the one launch
                # has no per-block counters): nominal exact projection 9 n^3 + n (n + 1) p flops, A read
                # and Pi written once
                nk, pk = self.cfg.sizes[self.ids[k]], res["npos"][j]
                infos[k] = {"iters": res["iters"][j], "status": 0 if st in (0, 3) else st, "npos": pk,
                            "err_bound": res["bound"][j], "path": "tiny-exact" if st == 3 else "tiny-lobpcg",
                            "flops": 9.0 * nk ** 3 + nk * (nk + 1.0) * pk, "bytes": 16.0 * nk * nk}
        t1 = time.perf_counter()
        if self.large:
            _, inf = api.project_batched(self.ctxs, [self.mats[k] for k in self.large], [tol] * len(self.large),
                                         outs=[self.outs[k] for k in self.large])
            for j, k in enumerate(self.large):
                infos[k] = dict(inf[j], path="direct" if inf[j].get("side") == 2 else "lobpcg")
        # host wall time of the two parts (each ends in a stream synchronisation)
        self.last_split_ms = (1e3 * (t1 - t0), 1e3 * (time.perf_counter() - t1))
        return infos

    def close(self):
        for c in self.ctxs:
            c.close()


def shard_c4(cfg, rank, world):
    costs = [block_cost(n, p) for n, p in zip(cfg.sizes, cfg.npos)]
    parts, loads = lpt_partition(costs, world)
    return parts[rank], loads


def run_c4(cfg, rank, world, dist, device, rounds, warmup, tol=None, tiny=True, paths=None, direct_n=0,
           params=None):
    """Sharded C4 rounds on this rank; returns (device ms of the timed rounds, max over ranks),
    projections done by all ranks, and the per-rank mean LOBPCG iterations. `paths` (a dict, if
    given) receives this rank's count of timed projections per path (lobpcg / direct / tiny-lobpcg /
    tiny-exact)."""
    import torch

    ids, _ = shard_c4(cfg, rank, world)
    sh = C4Shard(cfg, ids, device, tiny=tiny, direct_n=direct_n, params=params)
    st = torch.cuda.current_stream()
    for _ in range(warmup):
        sh.project(tol)
        sh.drift()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters, worst = [], 0
    ms = 0.0
    for _ in range(rounds):
        torch.cuda.synchronize()
        ev0.record(st)
        infos = sh.project(tol)
        ev1.record(st)
        torch.cuda.synchronize()
        ms += ev0.elapsed_time(ev1)
        iters += [i["iters"] for i in infos]
        worst = max([worst] + [i["status"] for i in infos])
        if paths is not None:
            for i in infos:
                paths[i["path"]] = paths.get(i["path"], 0) + 1
            work = paths.setdefault("alg_flops_bytes_per_round", [0.0, 0.0])
            work[0] += sum(i.get("flops", 0.0) for i in infos) / rounds
            work[1] += sum(i.get("bytes", 0.0) for i in infos) / rounds
            sp = paths.setdefault("host_ms_tiny_then_batched", [0.0, 0.0])
            sp[0] += sh.last_split_ms[0] / rounds
            sp[1] += sh.last_split_ms[1] / rounds
        sh.drift()  # the next round's inputs, outside the timed region
    if dist is not None:
        dist.barrier()
    t = torch.tensor([ms, float(len(ids) * rounds), float(worst)], dtype=torch.float64, device=device)
    if dist is not None:
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, proj, worst = float(mx[0]), float(sm[1]), int(mx[2])
    else:
        ms_max, proj = ms, float(len(ids) * rounds)
    sh.close()
    return ms_max, proj, (float(np.mean(iters)) if iters else 0.0), worst


def wall():
    return time.perf_counter()
