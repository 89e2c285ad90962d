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
