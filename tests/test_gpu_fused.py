"""GPU parity of the fused one-launch-per-image pipeline (csrc/pipe.cu):
preprocess + coarse-to-fine search of a batch of pairs, bit-exact against the
CPU oracle (tolerance 0: integer path) — offsets, every level's 9 candidate
errors, medians and every packed map of every image.  Calls go through the
C ABI (mtb_align_fused)."""

import numpy as np
import pytest

import mtb_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mtb(cuda):
    import paper_2007_06483_b200 as m
    from paper_2007_06483_b200 import _lib

    _lib.load()
    return m


def _stack(w, h, count, seed, max_shift):
    rng = np.random.default_rng(seed)
    base = np.dstack([orc.synthetic_gray(rng, w, h) for _ in range(3)])
    imgs, man = orc.generate_stack(base, count, seed=seed, max_shift=max_shift)
    return imgs, man


def _check(mtb, torch, imgs, pairs, levels=6, tol=4, maps=True):
    h, w = imgs[0].shape[:2]
    eng = mtb.MtbEngine(w, h, levels, tol)
    rgb = torch.from_numpy(np.stack(imgs)).cuda()
    pyr, acc, errs = eng.align_fused(rgb, pairs)
    torch.cuda.synchronize()
    pre = [orc.preprocess(im, levels, tol) for im in imgs]
    med = pyr.medians.cpu().numpy()
    for i, p in enumerate(pre):
        assert [lv["median"] for lv in p["mtb"]] == med[i].tolist(), i
        if maps:
            for k in range(eng.n):
                assert np.array_equal(eng.bitmap_words(pyr.mtb, i, k).cpu().numpy().view(np.uint64),
                                      orc.pack(p["mtb"][k]["mtb"])), (i, k)
                assert np.array_equal(eng.bitmap_words(pyr.excl, i, k).cpu().numpy().view(np.uint64),
                                      orc.pack(p["mtb"][k]["excl"])), (i, k)
    acc_h, errs_h = acc.cpu().numpy(), errs.cpu().numpy()
    for q, (r, t) in enumerate(pairs):
        want = orc.find_offset(pre[r]["mtb"], pre[t]["mtb"])
        assert tuple(acc_h[q, 0]) == tuple(want["offset"]), (q, acc_h[q, 0], want["offset"])
        for tr in want["traces"]:
            k = tr["level"]
            assert [e for _, e in tr["candidates"]] == errs_h[q, k].tolist(), (q, k)
            assert tuple(acc_h[q, k]) == tuple(tr["chosen"]), (q, k)
    return eng, pyr, acc, errs


@pytest.mark.parametrize("w,h,levels", [(512, 384, 6), (1008, 700, 6), (1024, 768, 6), (640, 480, 3),
                                        (64, 48, 6), (2000, 1004, 5)])
def test_fused_pairs_vs_oracle(mtb, cuda, w, h, levels):
    imgs, man = _stack(w, h, 4, seed=w + h, max_shift=min(20, w // 8))
    _check(mtb, cuda, imgs, [(0, 1), (2, 3)], levels=levels)


def test_fused_chain_and_pivot(mtb, cuda):
    imgs, man = _stack(768, 512, 5, seed=5, max_shift=12)
    chain = [(i, i + 1) for i in range(4)]
    _check(mtb, cuda, imgs, chain)
    pivot = [(2, i) for i in range(5) if i != 2]
    _check(mtb, cuda, imgs, pivot, maps=False)


def test_fused_config1_pairs(mtb, cuda):
    """Config 1 shape (1024x768, shifts up to the +-63 clamp), 8 pairs in one batch."""
    rng = np.random.default_rng(42)
    base = np.dstack([orc.synthetic_gray(rng, 1024, 768) for _ in range(3)])
    imgs, pairs, shifts = [], [], [(0, 0), (1, 0), (-5, 3), (63, -63), (-63, 63), (64, 0), (17, -9), (-2, 40)]
    for i, (dx, dy) in enumerate(shifts):
        a, _ = orc.generate_stack(base, 2, pairwise=[(dx, dy)], seed=i)
        imgs += a
        pairs.append((2 * i, 2 * i + 1))
    _check(mtb, cuda, imgs, pairs, maps=False)


def test_fused_degenerate(mtb, cuda):
    """Constant / black / white images give (0, 0) like test_search.py:65-72."""
    imgs = [np.full((96, 128, 3), v, np.uint8) for v in (0, 0, 255, 255, 77, 77)]
    _, _, acc, _ = _check(mtb, cuda, imgs, [(0, 1), (2, 3), (4, 5)])
    assert acc[:, 0].cpu().tolist() == [[0, 0]] * 3


def test_fused_matches_staged_24mp(mtb, cuda):
    """One full 6000x4000 pair: fused == staged engine (maps, medians, traces)."""
    torch = cuda
    from paper_2007_06483_b200.synth import apply_lut_device, synthetic_rgb_device, tone_lut
    from paper_2007_06483_b200.image import shift_rgb_device

    w, h = 6000, 4000
    eng = mtb.MtbEngine(w, h, 6, 4)
    base = synthetic_rgb_device(3, w, h)
    rgb = torch.empty((2, h, w, 3), dtype=torch.uint8, device="cuda")
    apply_lut_device(base, tone_lut(1.3, 0.9), out=rgb[0])
    moved = shift_rgb_device(base.unsqueeze(0), [(-37, 22)])[0]
    apply_lut_device(moved, tone_lut(0.7, 1.2), out=rgb[1])
    pyr_f, acc_f, errs_f = eng.align_fused(rgb, [(0, 1)])
    pyr_s = eng.preprocess(rgb)
    acc_s, errs_s = eng.search(pyr_s, [(0, 1)])
    torch.cuda.synchronize()
    assert torch.equal(pyr_f.medians, pyr_s.medians)
    for i in range(2):
        for k in range(eng.n):   # level views (arena padding words are never written)
            assert torch.equal(eng.bitmap_words(pyr_f.mtb, i, k), eng.bitmap_words(pyr_s.mtb, i, k)), (i, k)
            assert torch.equal(eng.bitmap_words(pyr_f.excl, i, k), eng.bitmap_words(pyr_s.excl, i, k)), (i, k)
    assert torch.equal(acc_f, acc_s) and torch.equal(errs_f, errs_s)


def test_fused_pair_patterns(mtb, cuda):
    """Two images per launch: pairs across launch boundaries, reversed pairs,
    self-pairs, repeated images and an odd image count (last launch has one
    K1 image)."""
    imgs, _ = _stack(512, 384, 7, seed=77, max_shift=16)
    pairs = [(1, 2), (2, 1), (6, 0), (3, 5), (0, 6), (4, 4), (5, 3), (0, 1), (6, 5), (2, 6)]
    _check(mtb, cuda, imgs, pairs, maps=True)


def test_fused_many_pairs_one_batch(mtb, cuda):
    """All 36 ordered-by-index pairs of 9 images in one call (many items per launch)."""
    imgs, _ = _stack(256, 192, 9, seed=91, max_shift=10)
    pairs = [(i, j) for i in range(9) for j in range(i + 1, 9)]
    _check(mtb, cuda, imgs, pairs, maps=False)


@pytest.mark.parametrize("w,h,n_img", [(16, 16, 1), (48, 20, 3), (512, 384, 1)])
def test_fused_preprocess_only_and_tiny(mtb, cuda, w, h, n_img):
    """No pairs (preprocess only), a single image, and the 16x16 minimum (one level)."""
    rs = np.random.RandomState(w * h + n_img)
    imgs = [rs.randint(0, 256, size=(h, w, 3), dtype=np.uint8) for _ in range(n_img)]
    _check(mtb, cuda, imgs, [], levels=6)
    if n_img >= 2:
        _check(mtb, cuda, imgs, [(0, n_img - 1)], levels=6)


@pytest.mark.parametrize("tol", [0, 127, 128, 200])
def test_fused_tolerances(mtb, cuda, tol):
    """Exclusion tolerance edge values (tol > 127 takes the generic compare)."""
    imgs, _ = _stack(512, 384, 2, seed=tol + 3, max_shift=9)
    _check(mtb, cuda, imgs, [(0, 1)], tol=tol)
