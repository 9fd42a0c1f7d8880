"""CPU, world_size 2 over gloo: the multi-rank batch path's host logic.

The GPU solve is replaced by a deterministic stand-in (the oracle's GS on
the rank's block), so what is tested here is exactly the part that runs on
the host: the block partition, one gather at the end, result order, and
bitwise independence of the partition.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1302_0120_b200.batch import BatchResult, shard_bounds, solve_batch_distributed
from paper_1302_0120_b200.patterns import make_problem
from paper_1302_0120_b200.solver import SolveConfig


def test_shard_bounds_cover_and_balance():
    for n in (0, 1, 7, 8, 256, 257):
        for world in (1, 2, 3, 4, 8):
            blocks = [shard_bounds(n, world, r) for r in range(world)]
            covered = [i for lo, hi in blocks for i in range(lo, hi)]
            assert covered == list(range(n))
            sizes = [hi - lo for lo, hi in blocks]
            assert max(sizes) <= -(-n // world)
    assert shard_bounds(256, 8, 7) == (224, 256)
    with pytest.raises(ValueError):
        shard_bounds(4, 2, 2)


def _oracle_stack(p, m_block, cfg, device):
    from oracle import phasemask_oracle as orc
    masks, gaps, its = [], [], []
    K = cfg.max_iters
    for m in m_block:
        o = orc.solve(p, m, K, cfg.precision.tag, record_every=cfg.record_every)
        masks.append(o["mask"])
        g = np.full(K, np.nan)
        for it, gap, _, _ in o["records"]:
            g[it - 1] = gap
        gaps.append(g)
        its.append(o["iters_run"])
    B = len(masks)
    shape = (B,) + p.shape
    nan = np.full((B, K), np.nan)
    return BatchResult(np.array(masks).reshape(shape), np.array(gaps).reshape(B, K), nan, nan.copy(),
                       np.array(its, dtype=np.int32), device_ms=1.0)


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, _ = make_problem(32, 3, 5)
        ms = np.stack([make_problem(32, 3, 100 + i)[1] for i in range(5)])
        cfg = SolveConfig(max_iters=4)
        res = solve_batch_distributed(p, ms, cfg, device=0, solve_fn=_oracle_stack)
        if rank == 0:
            out_q.put((res.phases, res.gap, res.iters_run))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_two_rank_gloo_batch_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    phases, gap, iters = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p, _ = make_problem(32, 3, 5)
    ms = np.stack([make_problem(32, 3, 100 + i)[1] for i in range(5)])
    ref = _oracle_stack(p, ms, SolveConfig(max_iters=4), 0)
    np.testing.assert_array_equal(phases, ref.phases)
    np.testing.assert_array_equal(gap, ref.gap)
    np.testing.assert_array_equal(iters, ref.iters_run)

