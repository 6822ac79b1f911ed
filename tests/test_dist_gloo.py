"""Multi-rank sharding logic on CPU: world_size 2 over gloo (127.0.0.1).

The engine's data-path collectives are (dist.py): an all-gather of each
rank's contiguous rows (labels, features, probe levels) and an all-reduce of
the zero-padded per-block pricing table.  Here the rank-local work is the CPU
oracle; the test checks that the gathered / reduced results equal the
single-rank ones bit for bit (the reference's determinism contract across
worker counts, cli.py:303-309).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_0805_1827_b200.dist import Shard
        from oracle import oracle as O
        from tests import _cases as CS
        shard = Shard(rank, world)
        p, s = CS.maxcall(5)
        mp_ = CS.packs(p, s)
        rp = CS.random_stumps(5, 9, 20, seed=1)
        ctx = O.Ctx(mp_, rp)
        # pricing: blocks sharded, zero-padded table all-reduced
        n_paths = 5 * 4096 + 77
        n_blocks = 6
        lo, hi = shard.range(n_blocks)
        table = torch.zeros((n_blocks, 3), dtype=torch.float64)
        if hi > lo:
            table[lo:hi] = torch.from_numpy(O.price_blocks(ctx, n_paths, 1827, lo, hi))
        shard.all_reduce_sum(table)
        # labels: rows gathered in rank order
        n = 13
        lo, hi = shard.range(n)
        pts = 100 * np.exp(0.2 * np.random.default_rng(0).normal(size=(n, 5)))
        keys = [O.derive_words(7, 2, i, 3) for i in range(n)]
        k = np.array([x[0] for x in keys]), np.array([x[1] for x in keys])
        local = torch.from_numpy(O.cmc_labels(ctx, pts[lo:hi], 3, 50, k[0][lo:hi], k[1][lo:hi], 10))
        gathered = shard.all_gather_rows(local, n)
        if rank == 0:
            q.put((table.numpy(), gathered.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sharding_is_bitwise_single_rank():
    from oracle import oracle as O
    from tests import _cases as CS
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    table, gathered = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p, s = CS.maxcall(5)
    mp_ = CS.packs(p, s)
    ctx = O.Ctx(mp_, CS.random_stumps(5, 9, 20, seed=1))
    full = O.price_blocks(ctx, 5 * 4096 + 77, 1827)
    assert np.array_equal(table, full)
    assert O.pool_moments(table[:, 0], table[:, 1], table[:, 2]) == O.pool_moments(full[:, 0], full[:, 1], full[:, 2])
    pts = 100 * np.exp(0.2 * np.random.default_rng(0).normal(size=(13, 5)))
    keys = [O.derive_words(7, 2, i, 3) for i in range(13)]
    ref = O.cmc_labels(ctx, pts, 3, 50, [x[0] for x in keys], [x[1] for x in keys], 10)
    assert np.array_equal(gathered, ref)
