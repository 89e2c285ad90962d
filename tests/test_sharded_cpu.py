"""Row-sharded single-pair alignment (config 5's decomposition) on CPU: the
orchestration of paper_2007_06483_b200/sharded.py driven through gloo with
2 and 3 ranks (and the in-process loopback) must reproduce the unsharded
oracle find_offset exactly — offsets and every level's 9 error counts."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import mtb_oracle as orc
from paper_2007_06483_b200.sharded import align_pair_distributed, align_pair_loopback, halo_sizes, plan_row_shards
from shard_oracle import OracleShard


def make_pair(seed, w, h, shift):
    rng = np.random.default_rng(seed)
    base = np.dstack([orc.smooth_gray(rng, w, h, cells=10) for _ in range(3)])
    imgs, man = orc.generate_stack(base, 2, pairwise=[shift], seed=seed)
    return imgs


def unsharded(imgs, levels):
    return orc.align_pairs(imgs, [(0, 1)], levels=levels)[0]


def same(res, want):
    assert tuple(res.offset) == tuple(want["offset"])
    for t, w in zip(res.traces, want["traces"]):
        assert t.level == w["level"] and tuple(t.chosen) == tuple(w["chosen"])
        assert [e for _, e in t.candidates] == [e for _, e in w["candidates"]]


def test_plan_row_shards_geometry():
    rows = plan_row_shards(25000, 10, 8)
    assert rows[0][0] == 0 and rows[-1][1] == 25000
    assert all(r0 % 512 == 0 for r0, _ in rows)
    assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
    assert [r1 - r0 for r0, r1 in rows] == [3072] * 7 + [3496]
    with pytest.raises(ValueError):
        plan_row_shards(1000, 10, 8)
    assert halo_sizes(0) == (1, 1) and halo_sizes(5) == (6, 0) and halo_sizes(-3) == (0, 4)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_loopback_matches_unsharded(world):
    imgs = make_pair(11 + world, 160, 200, (5, -7))
    res = align_pair_loopback(imgs[0], imgs[1], world, levels=4, shard_cls=OracleShard)
    same(res, unsharded(imgs, 4))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, imgs, levels, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h, w = imgs[0].shape[:2]
    n = min(levels, orc.max_levels(w, h))
    r0, r1 = plan_row_shards(h, n, world)[rank]
    res = align_pair_distributed(imgs[0][r0:r1], imgs[1][r0:r1], w, h, levels, shard_cls=OracleShard)
    out[rank] = (tuple(res.offset), [[e for _, e in t.candidates] for t in res.traces],
                 [tuple(t.chosen) for t in res.traces])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,shift", [(2, (9, 13)), (3, (-6, -11))])
def test_gloo_row_sharded_matches_unsharded(world, shift):
    imgs = make_pair(40 + world, 144, 256, shift)
    want = unsharded(imgs, 5)
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _port(), imgs, 5, out), nprocs=world, join=True)
        results = [out[r] for r in range(world)]
    for offset, errs, chosen in results:
        assert offset == tuple(want["offset"])
        assert errs == [[e for _, e in t["candidates"]] for t in want["traces"]]
        assert chosen == [tuple(t["chosen"]) for t in want["traces"]]
