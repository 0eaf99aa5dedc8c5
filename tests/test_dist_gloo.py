"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel host logic of
section 3.1: NCCL unique-id broadcast, max-over-ranks timing, per-rank data seeds,
per-job learning rate, arena sharding and the fixed summation tree of nnet_average,
emulated with gloo collectives and checked bit-exactly against the oracle average."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import training as otr
from paper_1410_7455_b200 import driver


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        uid = bytes(range(128)) if rank == 0 else None
        out["uid"] = driver.broadcast_bytes(uid)
        out["max"] = driver.max_over_ranks(float(rank + 3))
        # every job starts from the same model, trains on its own shard (seed per rank)
        rng = np.random.default_rng(driver.rank_seed(rank))
        count = 5_297_000 // 1000 + 17            # not a multiple of world or 64: ragged shards
        arena = rng.normal(size=count).astype(np.float32)
        # deterministic average: rank r reduces shard r of every rank in tree order
        gathered = [torch.zeros(count) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(arena))
        lo, hi = driver.shard_bounds(count, world, rank)
        shard = driver.shard_size(count, world)
        shards = [g.numpy()[lo:hi].astype(np.float32) for g in gathered]
        mine = np.zeros(shard, dtype=np.float32)            # padded shard (gather buffer layout)
        if hi > lo:
            mine[:hi - lo] = (driver.tree_reduce_stride(shards) * np.float32(1.0 / world)).astype(np.float32)
        pieces = [torch.zeros(shard) for _ in range(world)]
        dist.all_gather(pieces, torch.from_numpy(mine))
        out["avg"] = np.concatenate([p.numpy() for p in pieces]).astype(np.float32)[:count]
        out["all"] = [g.numpy().astype(np.float32) for g in gathered]
        out["lr"] = driver.job_learning_rate(0, 1, world)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multi_rank_average_and_helpers(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(res[r]["uid"] == bytes(range(128)) for r in range(world))
    assert all(res[r]["max"] == world + 2.0 for r in range(world))
    ref = otr.average_models([[a] for a in res[0]["all"]], dtype=np.float32)[0]
    for r in range(world):
        assert np.array_equal(res[r]["avg"], ref)                   # bit-exact vs oracle tree, every rank
    assert res[0]["lr"] == pytest.approx(0.01 * world / 6)          # lr x n_jobs / 6


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8])
def test_tree_schedule_matches_oracle_tree(n):
    rng = np.random.default_rng(n)
    vals = [rng.normal(size=33).astype(np.float32) for _ in range(n)]
    assert np.array_equal(driver.tree_reduce_stride(vals), otr.tree_sum(vals, np.float32))


def test_outer_iteration_sizes():
    mbs = driver.minibatches_per_outer_iteration(512)
    assert len(mbs) == 782 and sum(mbs) == 400_000 and mbs[-1] == 128     # reading R24
    assert driver.rank_seed(0) != driver.rank_seed(1)
    lo, hi = driver.shard_bounds(1024, 4, 3)
    assert (lo, hi) == (768, 1024)
    # the paper's 6 jobs on the config-3 arena (5 360 128 floats): ragged, covers everything
    count = 5_360_128
    b = [driver.shard_bounds(count, 6, r) for r in range(6)]
    assert b[0][0] == 0 and b[-1][1] == count and all(b[r][1] == b[r + 1][0] for r in range(5))
    assert driver.shard_size(count, 6) % 64 == 0


def test_block_randomize_matches_oracle_and_partitions_jobs():
    """driver.block_randomize (the product's data schedule) against the oracle's C.2 blocks:
    same examples in every block (the product uses balanced integer cut points, the oracle
    numpy.array_split: equal sizes up to one), disjoint across jobs."""
    from oracle import data as odata
    for F, N, K in [(10_000, 1, 400), (100_003, 4, 3000), (262_144, 8, 32_768)]:
        a = driver.block_randomize(F, N, K, seed=11)
        b = odata.block_randomize(F, N, K, seed=11)
        assert len(a) == len(b) == N
        flat_a = np.concatenate([blk for row in a for blk in row])
        flat_b = np.concatenate([blk for row in b for blk in row])
        assert np.array_equal(np.sort(flat_a), np.arange(F)) and np.array_equal(flat_a, flat_b)
        assert max(len(x) for row in a for x in row) - min(len(x) for row in a for x in row) <= 1
