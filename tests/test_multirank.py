"""Batch sharding across ranks on CPU (gloo, world size 2): every pair is
owned by exactly one rank, results gathered from the shards equal the
single-process results, and the job time is the max over ranks."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import mtb_oracle as orc
from paper_2007_06483_b200.dist import max_over_ranks, shard_pairs, shard_range, sum_over_ranks


@pytest.mark.parametrize("n,world", [(0, 2), (1, 2), (7, 2), (16, 8), (4096, 8), (5, 3)])
def test_shard_range_partitions(n, world):
    seen = []
    for r in range(world):
        b, e = shard_range(n, r, world)
        assert 0 <= b <= e <= n
        seen.extend(range(b, e))
    assert seen == list(range(n))
    sizes = [shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, pairs, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard_pairs(pairs, rank, world)
    # each rank aligns its own pairs (here with the CPU oracle, standing in for
    # the device engine; the host logic under test is the sharding/timing)
    offs = []
    for seed in mine:
        rng = np.random.default_rng(seed)
        base = np.dstack([orc.smooth_gray(rng, 96, 80) for _ in range(3)])
        imgs, man = orc.generate_stack(base, 2, seed=seed, max_shift=5)
        offs.append((seed, orc.align_pairs(imgs, [(0, 1)], levels=3)[0]["offset"]))
    t = max_over_ranks(0.1 * (rank + 1))
    total = sum_over_ranks(len(mine))
    gathered = [None] * world
    dist.all_gather_object(gathered, offs)
    if rank == 0:
        results["t"] = t
        results["total"] = total
        results["offs"] = [o for part in gathered for o in part]
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_batch_shard_matches_single_process():
    pairs = list(range(11))
    port = _free_port()
    with mp.Manager() as m:
        results = m.dict()
        mp.spawn(_worker, args=(2, port, pairs, results), nprocs=2, join=True)
        got = dict(results["offs"])
        assert results["total"] == len(pairs)
        assert abs(results["t"] - 0.2) < 1e-12
    for seed in pairs:
        rng = np.random.default_rng(seed)
        base = np.dstack([orc.smooth_gray(rng, 96, 80) for _ in range(3)])
        imgs, man = orc.generate_stack(base, 2, seed=seed, max_shift=5)
        assert tuple(got[seed]) == tuple(orc.align_pairs(imgs, [(0, 1)], levels=3)[0]["offset"])
