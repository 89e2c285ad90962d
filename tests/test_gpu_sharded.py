"""Row-sharded single-pair alignment on the GPU (config 5's decomposition),
with W virtual shards on one device (loopback driver, the same CudaShard
phases as the NCCL path): bit-identical to the unsharded engine — offset and
every level's 9 error counts — including 10-level pyramids."""

import numpy as np
import pytest

import mtb_oracle as orc

pytestmark = pytest.mark.gpu


def _unsharded(mtb, cuda, imgs, levels):
    from paper_2007_06483_b200.engine import results_from_device

    h, w = imgs[0].shape[:2]
    eng = mtb.MtbEngine(w, h, levels, 4)
    pyr = eng.preprocess(cuda.from_numpy(np.stack(imgs)).cuda())
    acc, errs = eng.search(pyr, [(0, 1)])
    return results_from_device(acc, errs)[0]


def _same(a, b):
    assert tuple(a.offset) == tuple(b.offset)
    for ta, tb in zip(a.traces, b.traces):
        assert ta.level == tb.level and ta.chosen == tb.chosen
        assert [e for _, e in ta.candidates] == [e for _, e in tb.candidates]


@pytest.fixture(scope="module")
def mtb(cuda):
    import paper_2007_06483_b200 as m

    return m


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_loopback_matches_unsharded_6_levels(mtb, cuda, world):
    from paper_2007_06483_b200.sharded import align_pair_loopback

    rng = np.random.default_rng(20 + world)
    base = np.dstack([orc.synthetic_gray(rng, 1000, 768) for _ in range(3)])
    imgs, man = orc.generate_stack(base, 2, seed=world, max_shift=40)
    res = align_pair_loopback(imgs[0], imgs[1], world, levels=6)
    _same(res, _unsharded(mtb, cuda, imgs, 6))
    # and against the CPU oracle
    want = orc.align_pairs(imgs, [(0, 1)], levels=6)[0]
    assert tuple(res.offset) == tuple(want["offset"])


@pytest.mark.parametrize("world", [4, 8])
def test_loopback_10_levels(mtb, cuda, world):
    """8448 x 8192 (10 levels, level 9 is 16 x 16), shifts beyond 64 px."""
    from paper_2007_06483_b200.sharded import align_pair_loopback
    from paper_2007_06483_b200.synth import synthetic_rgb_device
    from paper_2007_06483_b200.image import shift_rgb_device

    torch = cuda
    w, h = 8448, 8192
    base = synthetic_rgb_device(77, w, h)
    moved = shift_rgb_device(base.unsqueeze(0), [(150, -90)])[0]
    imgs = [base.cpu().numpy(), moved.cpu().numpy()]
    res = align_pair_loopback(imgs[0], imgs[1], world, levels=10)
    ref = _unsharded(mtb, torch, imgs, 10)
    _same(res, ref)
    assert len(res.traces) == 10


def test_level_loop_has_no_host_sync(mtb, cuda):
    """The row-sharded level loop (halo views, 3-segment counts, sums, device
    decisions) runs under torch's sync debug mode "error": no host round trip
    between levels."""
    from paper_2007_06483_b200.sharded import CudaShard, loopback_levels, pair_levels, plan_row_shards

    rng = np.random.default_rng(5)
    base = np.dstack([orc.synthetic_gray(rng, 1024, 1024) for _ in range(3)])
    imgs, _ = orc.generate_stack(base, 2, seed=5, max_shift=30)
    h, w = imgs[0].shape[:2]
    n = pair_levels(w, h, 6)
    shards = [CudaShard(w, h, r0, r1, n) for r0, r1 in plan_row_shards(h, n, 4)]
    hists = [sh.preprocess(sh.stack_rows(imgs[0][r0:r1], imgs[1][r0:r1]))
             for sh, (r0, r1) in zip(shards, plan_row_shards(h, n, 4))]
    ghist = sum(hists[1:], hists[0])
    for sh in shards:
        sh.threshold(ghist)
    cuda.cuda.synchronize()
    cuda.cuda.set_sync_debug_mode("error")
    try:
        accs, errs = loopback_levels(shards, n)
    finally:
        cuda.cuda.set_sync_debug_mode("default")
    want = orc.align_pairs(imgs, [(0, 1)], levels=6)[0]
    assert tuple(accs[0][0].tolist()) == tuple(want["offset"])


def _nccl_worker(rank, world, port, w, h, out):
    import os

    import torch
    import torch.distributed as dist

    from paper_2007_06483_b200.sharded import align_pair_distributed, pair_levels, plan_row_shards
    from paper_2007_06483_b200.synth import generate_stack, synthetic_rgb_device

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    imgs, _ = generate_stack(synthetic_rgb_device(12, w, h), 2, seed=12, max_shift=60)
    n = pair_levels(w, h, 10)
    r0, r1 = plan_row_shards(h, n, world)[rank]
    res = align_pair_distributed(imgs[0][r0:r1].contiguous(), imgs[1][r0:r1].contiguous(), w, h, 10)
    out[rank] = (tuple(res.offset), [[e for _, e in t.candidates] for t in res.traces])
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_row_sharded_when_two_gpus(mtb, cuda):
    """align_pair_distributed with CudaShard over NCCL (batched neighbour P2P
    halos, 9-count all-reduces) equals the unsharded engine; needs >= 2 GPUs."""
    if cuda.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import socket

    import torch.multiprocessing as mp

    from paper_2007_06483_b200.synth import generate_stack, synthetic_rgb_device

    w, h = 4096, 4096
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_nccl_worker, args=(2, port, w, h, out), nprocs=2, join=True)
        got = [out[r] for r in range(2)]
    imgs, _ = generate_stack(synthetic_rgb_device(12, w, h), 2, seed=12, max_shift=60)
    ref = _unsharded(mtb, cuda, [im.cpu().numpy() for im in imgs], 10)
    for offset, errs in got:
        assert offset == tuple(ref.offset)
        assert errs == [[e for _, e in t.candidates] for t in ref.traces]
