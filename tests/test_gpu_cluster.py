"""On-chip small-image preprocess (csrc/cluster.cu, `mtb_preprocess_maps`):
each image's gray pyramid lives in a thread-block cluster's shared memory.

Bit-exact (integer path, tolerance 0) against the staged kernels (K1 +
hist_median + threshold, themselves oracle-checked) over a spread of
geometries that exercise every cluster size, partial edge tiles, padding
words, levels 4-5 words spanning tiles of different CTAs and 1-6 levels, and
directly against the CPU oracle (oracle/mtb_oracle.py) for config 1's shape
(1024 x 768, 6 levels) including the search traces.
"""

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


def _batch(cuda, w, h, n, seed):
    from paper_2007_06483_b200.synth import synthetic_rgb_device

    return cuda.stack([synthetic_rgb_device(seed + i, w, h) for i in range(n)]).contiguous()


def _same_as_staged(mtb, cuda, w, h, levels, tol, n=5, seed=0):
    eng = mtb.MtbEngine(w, h, levels, tol)
    assert eng.maps_cluster() > 0, (w, h, levels)
    batch = _batch(cuda, w, h, n, seed)
    want = eng.preprocess(batch, keep_hist=True)
    got = eng.alloc(n, keep_hist=True, gray=False)
    eng.preprocess_maps(batch, got)
    cuda.cuda.synchronize()
    assert cuda.equal(got.medians, want.medians), (w, h)
    assert cuda.equal(got.hist, want.hist), (w, h)
    for i in range(n):
        for k in range(eng.n):
            assert cuda.equal(eng.bitmap_words(got.mtb, i, k), eng.bitmap_words(want.mtb, i, k)), (w, h, i, k)
            assert cuda.equal(eng.bitmap_words(got.excl, i, k), eng.bitmap_words(want.excl, i, k)), (w, h, i, k)
    return eng


@pytest.mark.parametrize("w,h,levels,tol", [
    (1024, 768, 6, 4),      # config 1
    (640, 480, 6, 4),
    (1504, 1000, 6, 4),     # 6 x 32 tiles: the largest shapes need 16-CTA clusters
    (336, 200, 6, 0),       # partial tiles both ways, tol 0
    (1040, 770, 5, 200),    # odd tile counts, level-3 padding word, 5 levels, wide tolerance
    (96, 64, 3, 4),         # one tile, 3 levels
    (2048, 96, 6, 4),       # short and wide: fewer tiles than CTAs in some clusters
    (16, 16, 1, 4),         # smallest legal image, 1 level
])
def test_maps_equal_staged(mtb, cuda, w, h, levels, tol):
    _same_as_staged(mtb, cuda, w, h, levels, tol)


def test_every_cluster_size(mtb, cuda, monkeypatch):
    """Force each cluster size and group count the selector may pick."""
    from paper_2007_06483_b200 import _lib

    for c, g in [(1, 4), (2, 3), (4, 2), (8, 3), (16, 4)]:
        monkeypatch.setenv("MTB_CM_CLUSTER", str(c))
        monkeypatch.setenv("MTB_CM_GROUPS", str(g))
        w, h = (256, 192) if c == 1 else (512, 384) if c < 8 else (1024, 768)
        if int(_lib.load().mtb_preprocess_maps_cluster(w, h, 6)) != c:
            continue   # shape does not fit that cluster on this device
        _same_as_staged(mtb, cuda, w, h, 6, 4, n=3, seed=10 * c + g)


def test_config1_vs_oracle_with_search(mtb, cuda):
    """1024 x 768 pairs (config 1): medians, maps and search traces vs the oracle."""
    from paper_2007_06483_b200.synth import generate_stack, synthetic_rgb_device

    w, h = 1024, 768
    eng = mtb.MtbEngine(w, h, 6, 4)
    imgs = []
    for s in range(3):
        st, _ = generate_stack(synthetic_rgb_device(70 + s, w, h), 2, seed=70 + s, max_shift=63)
        imgs += st
    batch = cuda.stack(imgs).contiguous()
    pyr = eng.alloc(len(imgs), gray=False)
    eng.preprocess_maps(batch, pyr)
    pairs = [(0, 1), (2, 3), (4, 5)]
    acc, errs = eng.search(pyr, pairs)
    med = pyr.medians.cpu().numpy()
    acc_h, errs_h = acc.cpu().numpy(), errs.cpu().numpy()
    pre = []
    for i, im in enumerate(imgs):
        p = orc.preprocess(im.cpu().numpy(), 6, 4)
        pre.append(p)
        assert [lv["median"] for lv in p["mtb"]] == med[i].tolist(), i
        for k in range(eng.n):
            assert np.array_equal(eng.bitmap_words(pyr.mtb, i, k).cpu().numpy().view(np.uint64),
                                  orc.pack(p["mtb"][k]["mtb"])), (i, k)
            assert np.array_equal(eng.bitmap_words(pyr.excl, i, k).cpu().numpy().view(np.uint64),
                                  orc.pack(p["mtb"][k]["excl"])), (i, k)
    for q, (r, t) in enumerate(pairs):
        want = orc.find_offset(pre[r]["mtb"], pre[t]["mtb"])
        assert tuple(acc_h[q, 0]) == tuple(want["offset"]), q
        for tr in want["traces"]:
            assert [e for _, e in tr["candidates"]] == errs_h[q, tr["level"]].tolist(), (q, tr["level"])


def test_unsupported_shapes_are_refused(mtb, cuda):
    from paper_2007_06483_b200 import _lib

    lib = _lib.load()
    assert lib.mtb_preprocess_maps_cluster(6000, 4000, 6) == 0     # does not fit a cluster
    assert lib.mtb_preprocess_maps_cluster(1024, 1024, 7) == 0     # more than 6 levels
    eng = mtb.MtbEngine(6000, 4000, 6, 4)
    assert eng.maps_cluster() == 0
    batch = cuda.zeros((1, 4000, 6000, 3), dtype=cuda.uint8, device="cuda")
    pyr = eng.alloc(1, gray=False)
    with pytest.raises(ValueError):
        eng.preprocess_maps(batch, pyr)


def test_many_images_one_launch(mtb, cuda):
    """More images than clusters (persistent loop, triple-buffered sums)."""
    from paper_2007_06483_b200 import _lib

    w, h, n = 256, 192, 300
    eng = mtb.MtbEngine(w, h, 6, 4)
    batch = _batch(cuda, w, h, n, 5)
    want = eng.preprocess(batch)
    got = eng.alloc(n, gray=False)
    before = _lib.load().mtb_launch_count()
    eng.preprocess_maps(batch, got)
    assert _lib.load().mtb_launch_count() - before == 1
    assert cuda.equal(got.medians, want.medians)
    for k in range(eng.n):
        nw64, off = int(eng.geom[k, 4]), int(eng.geom[k, 5])
        sl = slice(off, off + nw64 * int(eng.geom[k, 1]))
        assert cuda.equal(got.mtb[:, sl], want.mtb[:, sl]), k
        assert cuda.equal(got.excl[:, sl], want.excl[:, sl]), k


def test_dispatch_by_cluster_size(mtb, cuda):
    """preprocess(maps_only=True) takes the on-chip kernel only where it is
    faster (clusters of <= 2 CTAs); the drop-in API results are the same."""
    small = mtb.MtbEngine(512, 384, 6, 4)
    assert small.maps_cluster() in (1, 2) and small.on_chip_maps()
    batch = _batch(cuda, 512, 384, 4, 3)
    pyr = small.preprocess(batch, maps_only=True)
    assert pyr.gray is None
    want = small.preprocess(batch)
    assert cuda.equal(pyr.medians, want.medians)
    big = mtb.MtbEngine(1024, 768, 6, 4)
    assert big.maps_cluster() > 2 and not big.on_chip_maps()
    assert big.preprocess(_batch(cuda, 1024, 768, 2, 3), maps_only=True).gray is not None
    imgs = [batch[i].cpu().numpy() for i in range(4)]
    off = mtb.get_exp_shift(imgs[0], imgs[1])
    pre = [orc.preprocess(im, 6, 4) for im in imgs[:2]]
    assert tuple(off) == tuple(orc.find_offset(pre[0]["mtb"], pre[1]["mtb"])["offset"])


def test_dense_histograms_match_spread(mtb, cuda):
    """mtb_preprocess switches to dense staged histograms when each K1 CTA
    covers >= 2 whole images (n_img >= 2 x SMs); level 6 comes from the
    tail pyramid pass, which flush with the same stride.  Medians, dense
    histograms and maps equal the split entry points (spread layout)."""
    w = h = 1024
    n = 300
    eng = mtb.MtbEngine(w, h, 7, 4)
    assert eng.n == 7
    batch = _batch(cuda, w, h, 8, 21).repeat(n // 8 + 1, 1, 1, 1)[:n].contiguous()
    dense = eng.preprocess(batch, keep_hist=True)          # one mtb_preprocess call: dense bins
    spread = eng.alloc(n, keep_hist=True)
    for i0 in range(0, n, 100):                             # K1 launches of 100 images: spread bins
        eng.pyramid_hist(batch, spread, i0, 100)
    eng.threshold_levels(spread, n)                         # one median pass, layout read per image
    split_dense = eng.alloc(n, keep_hist=True)
    eng.pyramid_hist(batch, split_dense)                    # one K1 launch of 300: dense bins
    eng.threshold_levels(split_dense, n)
    assert cuda.equal(split_dense.medians, spread.medians)
    assert cuda.equal(dense.medians, spread.medians)
    assert cuda.equal(dense.hist, spread.hist)
    for k in range(eng.n):
        nw64, off = int(eng.geom[k, 4]), int(eng.geom[k, 5])
        sl = slice(off, off + nw64 * int(eng.geom[k, 1]))
        assert cuda.equal(dense.mtb[:, sl], spread.mtb[:, sl]), k
        assert cuda.equal(dense.excl[:, sl], spread.excl[:, sl]), k
    host = batch[0].cpu().numpy()
    want = orc.preprocess(host, 7, 4)
    assert [lv["median"] for lv in want["mtb"]] == dense.medians[0].tolist()
