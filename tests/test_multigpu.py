"""Batch sharding across ranks (BASELINE configs[3]): LPT partition properties and a
world_size-2 gloo run of the host-side sharding + scalar reductions (no GPU needed)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1912_02767_b200.multigpu import block_cost, lpt_bound, lpt_partition, shard_c4
from workloads.generators import C4


def test_lpt_partition_covers_and_balances():
    cfg = C4()
    costs = [block_cost(n, p) for n, p in zip(cfg.sizes, cfg.npos)]
    for world in (1, 2, 3, 4, 8):
        parts, loads = lpt_partition(costs, world)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(costs)))          # every block exactly once
        assert max(loads) <= lpt_bound(costs, world) + 1e-6 * sum(costs)
        assert parts == lpt_partition(costs, world)[0]  # deterministic


def test_lpt_small_exact():
    # 2 ranks, costs 5,4,3,3,3 -> LPT: r0 {5,3}, r1 {4,3,3}? LPT gives 5|4, 3->r1(4), 3->r0(5)... loads 8|10
    parts, loads = lpt_partition([5.0, 4.0, 3.0, 3.0, 3.0], 2)
    assert sorted(loads) == [8.0, 10.0]
    assert sorted(parts, key=len) == [[0, 3], [1, 2, 4]] or sorted(parts, key=len) == [[0, 2], [1, 3, 4]]


def test_block_cost_direct_branch():
    assert block_cost(300, 150) == 300.0 ** 3 / 8.0          # min(p, n-p) >= n/3: DIRECT
    assert block_cost(300, 20) == 300.0 ** 2 * (20 + 16)    # LOBPCG on the smaller side


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = C4()
    ids, loads = shard_c4(cfg, rank, world)
    got = [None] * world
    dist.all_gather_object(got, ids)
    # per-round scalars as run_c4 reduces them: max device time, sum of projections, worst status
    t = torch.tensor([10.0 + rank, float(len(ids)), float(rank % 2)], dtype=torch.float64)
    mx, sm = t.clone(), t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    if rank == 0:
        out.put((got, mx.tolist(), sm.tolist(), loads))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharding():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, mx, sm, loads = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(got[0] + got[1]) == list(range(512))
    assert not set(got[0]) & set(got[1])
    assert mx[0] == 11.0 and sm[1] == 512.0 and mx[2] == 1.0
    assert max(loads) / min(loads) < 1.01   # 512 blocks balance to well under 1%


# ---------------------------------------------------------------- row-sharded single matrix (§8.e)
def test_row_blocks_partition():
    from paper_1912_02767_b200.api import row_blocks
    for n, world in ((4000, 8), (4001, 3), (7, 4), (5, 5)):
        blocks = row_blocks(n, world)
        assert blocks[0][0] == 0 and sum(r for _, r in blocks) == n
        assert all(blocks[k + 1][0] == blocks[k][0] + blocks[k][1] for k in range(world - 1))
        assert max(r for _, r in blocks) - min(r for _, r in blocks) <= 1


def _gram_worker(rank, world, port, out):
    """Host reference of the sharded math the library runs over NCCL: every Gram S^T (B S) is the
    sum of the row-block partials, the column norms are sums of squares, and the gathered block
    multiply A_local Z_full equals the row block of A Z."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1912_02767_b200.api import row_blocks
    rng = np.random.default_rng(0)
    n, s = 97, 11
    M = rng.standard_normal((n, n))
    A = (M + M.T) / 2
    S = rng.standard_normal((n, s))
    r0, nr = row_blocks(n, world)[rank]
    Sl = S[r0:r0 + nr]
    # all-gather of the local rows (rank order) -> full S; A_local S_full = rows of A S
    parts = [None] * world
    dist.all_gather_object(parts, Sl)
    Sfull = np.vstack(parts)
    Yl = A[r0:r0 + nr] @ Sfull
    G = torch.from_numpy(Sl.T @ Yl)
    dist.all_reduce(G)
    cn = torch.from_numpy((Sl ** 2).sum(axis=0))
    dist.all_reduce(cn)
    if rank == 0:
        out.put((G.numpy(), np.sqrt(cn.numpy()), S.T @ (A @ S), np.linalg.norm(S, axis=0)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharded_gram_identity():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gram_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    G, cn, Gref, cnref = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.abs(G - Gref).max() <= 1e-12 * np.abs(Gref).max()
    assert np.abs(cn - cnref).max() <= 1e-13 * cnref.max()
