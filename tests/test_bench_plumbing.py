"""CPU checks of bench.py's workload plumbing (configs, pair lists) and of the
row-shard halo geometry."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_unit_pairs_and_configs():
    import bench

    assert bench.unit_pairs(3, 2) == [(0, 1), (2, 3), (4, 5)]
    p = bench.unit_pairs(2, 7)
    assert p[:6] == [(3, 0), (3, 1), (3, 2), (3, 4), (3, 5), (3, 6)] and p[6] == (10, 7) and len(p) == 12
    assert {c: (v["width"], v["height"]) for c, v in bench.CONFIGS.items()} == {
        1: (1024, 768), 2: (6000, 4000), 3: (6000, 4000), 4: (4000, 3000)}


def test_halo_rows_cover_every_reachable_base():
    """halo_rows(n, k) bounds |base dy| + 1 for every offset the coarse-to-fine
    search can reach (search.py:85-95: base = 2 * previous choice, choice =
    base + {-1, 0, 1}); plan_row_shards keeps it below any shard's rows."""
    from paper_2007_06483_b200.sharded import halo_rows, level_rows, plan_row_shards

    for n in range(1, 11):
        reach = {0}
        for k in reversed(range(n)):
            bases = {2 * d for d in reach} if k < n - 1 else {0}
            assert max(abs(b) for b in bases) + 1 <= halo_rows(n, k)
            reach = {b + e for b in bases for e in (-1, 0, 1)}
    for world in (2, 3, 8):
        rows = plan_row_shards(25000, 10, world)
        for k in range(10):
            assert all(level_rows(r0, r1, k)[1] - level_rows(r0, r1, k)[0] > halo_rows(10, k) for r0, r1 in rows)
    with pytest.raises(ValueError):
        plan_row_shards(25000, 10, 25)   # 48 blocks < 2 per shard


def test_bench_dispatch_threshold_matches_the_product():
    import bench
    from paper_2007_06483_b200 import pipeline

    assert bench.FUSED_MIN_PIXELS == pipeline.FUSED_MIN_PIXELS
    assert bench.FUSED_MIN_IMAGES == pipeline.FUSED_MIN_IMAGES
    cfg = bench.CONFIGS
    assert bench.fused_default(cfg[2]["width"], cfg[2]["height"], cfg[2]["units"] * cfg[2]["stack"])
    assert bench.fused_default(cfg[3]["width"], cfg[3]["height"], cfg[3]["units"] * cfg[3]["stack"])
    assert not bench.fused_default(cfg[4]["width"], cfg[4]["height"], cfg[4]["units"] * cfg[4]["stack"])
    assert not bench.fused_default(cfg[1]["width"], cfg[1]["height"], cfg[1]["units"] * cfg[1]["stack"])
