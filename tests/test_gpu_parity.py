"""GPU parity: the sm_100a path against the reference's golden vectors and
the CPU oracle, bit-exact (all integer arithmetic, so the tolerance is 0).

Every call here goes through the C ABI (paper_2007_06483_b200/_lib.py ->
libmtbalign_b200.so).  Run on a B200 with `pytest -m gpu`.
"""

import hashlib

import numpy as np
import pytest

import mtb_oracle as orc

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def mtb(cuda):
    import paper_2007_06483_b200 as m
    from paper_2007_06483_b200 import _lib

    _lib.load()
    return m


# ----------------------------------------------------------- known answers --
def test_known_answers(mtb):
    assert mtb.to_grayscale(np.array([[[255, 0, 0]]], np.uint8))[0, 0] == 53
    assert (mtb.to_grayscale(np.full((2, 3, 3), 255, np.uint8)) == 255).all()
    assert mtb.downsample_half(np.array([[0, 0], [255, 255]], np.uint8))[0, 0] == 128
    lv = mtb.build_pyramid(np.zeros((1440, 2560), np.uint8), 6)
    assert len(lv) == 6 and lv[-1].shape == (45, 80)
    img = np.zeros((64, 64), np.uint8)
    lv = mtb.build_pyramid(img, 6)
    assert len(lv) == 3 and lv[-1].shape == (16, 16) and lv[0] is img
    assert mtb.median_from_histogram(mtb.histogram(np.array([[0, 1], [2, 3]], np.uint8))) == 1
    assert mtb.median_from_histogram(mtb.histogram(np.array([[0, 255]] * 8, np.uint8))) == 0
    ramp = np.repeat(np.arange(256, dtype=np.uint8), 4).reshape(32, 32)
    assert mtb.median_from_histogram(mtb.histogram(ramp)) == 127
    assert mtb.make_mtb(ramp, 127).count_ones() == 512
    eb = mtb.make_exclusion(np.array([[100, 104, 105, 96, 95]], np.uint8), 100, 4)
    assert eb.to_bool().tolist() == [[False, False, True, False, True]]
    assert mtb.make_exclusion(np.array([[0]], np.uint8), 2, 4).count_ones() == 0
    assert mtb.make_exclusion(np.array([[255]], np.uint8), 253, 4).count_ones() == 0
    with pytest.raises(ValueError):
        mtb.median_from_histogram(np.zeros(256, np.int64))
    for w in (1, 31, 63, 64, 65, 127, 128, 129):
        b = mtb.Bitmap.from_bool(np.ones((3, w), bool))
        assert b.count_ones() == 3 * w and int(np.bitwise_count(b.buf).sum()) == 3 * w
    assert mtb.Bitmap.from_bool(np.ones((3, 7), bool), "bytemap").count_ones() == 21


def test_bitmap_views_match_reference_layout(mtb):
    rs = np.random.RandomState(11)
    mask = rs.rand(9, 131) < 0.4
    p = mtb.Bitmap.from_bool(mask, "packed")
    assert np.array_equal(p.buf, orc.pack(mask))
    assert np.array_equal(p.to_bool(), mask)
    b = mtb.Bitmap.from_bool(mask, "bytemap")
    assert set(np.unique(b.buf).tolist()) <= {0, 255}
    assert np.array_equal(b.buf != 0, mask)
    for y in range(9):
        for x in range(0, 131, 7):
            assert p.get(x, y) == bool(mask[y, x]) == b.get(x, y)
    with pytest.raises(IndexError):
        p.get(131, 0)


# ------------------------------------------------------ golden: primitives --
def test_gray_golden(mtb, golden):
    _, arr = golden
    assert np.array_equal(mtb.to_grayscale(arr["gray_in"]), arr["gray_out"])
    assert np.array_equal(mtb.to_grayscale(arr["gray_solid_in"]), arr["gray_solid_out"])


def test_api_pyramid_threshold_golden(mtb, golden):
    meta, arr = golden
    for ci, case in enumerate(meta["pyramid_cases"]):
        img = arr[f"pyr{ci}_in"]
        levels = mtb.build_pyramid(img, case["levels_requested"])
        pairs = mtb.build_mtb_pyramid(levels, case["tol"])
        assert len(levels) == case["n"]
        for k, (lv, pr) in enumerate(zip(levels, pairs)):
            assert np.array_equal(lv, arr[f"pyr{ci}_l{k}"]), (ci, k)
            assert np.array_equal(mtb.histogram(lv), arr[f"pyr{ci}_h{k}"])
            assert pr.median == case["medians"][k]
            assert np.array_equal(pr.mtb.buf, arr[f"pyr{ci}_m{k}"]), (ci, k)
            assert np.array_equal(pr.exclusion.buf, arr[f"pyr{ci}_e{k}"]), (ci, k)


def test_fused_engine_golden(mtb, golden, cuda):
    """Fused preprocess (RGB with R=G=B so gray == the golden input)."""
    meta, arr = golden
    for ci, case in enumerate(meta["pyramid_cases"]):
        g = arr[f"pyr{ci}_in"]
        rgb = cuda.from_numpy(np.repeat(g[:, :, None], 3, axis=2)).cuda().unsqueeze(0).contiguous()
        eng = mtb.MtbEngine(case["w"], case["h"], case["levels_requested"], case["tol"])
        pyr = eng.preprocess(rgb, keep_hist=True)
        assert eng.n == case["n"]
        med = pyr.medians.cpu().numpy()[0]
        hist = pyr.hist.cpu().numpy()[0]
        for k in range(eng.n):
            assert np.array_equal(eng.gray_level(pyr, 0, k).cpu().numpy(), arr[f"pyr{ci}_l{k}"]), (ci, k)
            assert np.array_equal(hist[k].astype(np.int64), arr[f"pyr{ci}_h{k}"]), (ci, k)
            assert med[k] == case["medians"][k]
            assert np.array_equal(eng.bitmap_words(pyr.mtb, 0, k).cpu().numpy().view(np.uint64),
                                  arr[f"pyr{ci}_m{k}"]), (ci, k)
            assert np.array_equal(eng.bitmap_words(pyr.excl, 0, k).cpu().numpy().view(np.uint64),
                                  arr[f"pyr{ci}_e{k}"]), (ci, k)


@pytest.mark.parametrize("w,h,L", [(16, 16, 6), (17, 19, 6), (100, 37, 6), (129, 64, 6), (200, 150, 6),
                                   (1023, 769, 6), (777, 1030, 6), (2100, 1500, 10), (1024, 768, 6),
                                   (333, 4100, 9), (4100, 70, 3)])
def test_fused_engine_vs_oracle(mtb, cuda, w, h, L):
    """Odd widths (scalar RGB path), unaligned pitches, deep pyramids (second tile pass)."""
    rs = np.random.RandomState(w * 7 + h)
    rgb = rs.randint(0, 256, size=(2, h, w, 3), dtype=np.uint8)
    rgb[1] = np.clip(rgb[1].astype(np.int32) * 2 - 100, 0, 255)   # saturated exposure
    eng = mtb.MtbEngine(w, h, L, 4)
    pyr = eng.preprocess(cuda.from_numpy(rgb).cuda(), keep_hist=True)
    med = pyr.medians.cpu().numpy()
    for i in range(2):
        want = orc.preprocess(rgb[i], L, 4)
        assert eng.n == len(want["pyramid"])
        for k in range(eng.n):
            lv = want["pyramid"][k]
            assert np.array_equal(eng.gray_level(pyr, i, k).cpu().numpy(), lv), (i, k)
            assert med[i, k] == want["mtb"][k]["median"]
            assert np.array_equal(eng.bitmap_words(pyr.mtb, i, k).cpu().numpy().view(np.uint64),
                                  orc.pack(want["mtb"][k]["mtb"])), (i, k)
            assert np.array_equal(eng.bitmap_words(pyr.excl, i, k).cpu().numpy().view(np.uint64),
                                  orc.pack(want["mtb"][k]["excl"])), (i, k)


# ------------------------------------------------------ golden: error test --
def test_shifted_error_golden(mtb, golden):
    meta, arr = golden
    eng = mtb.kernels.active()
    for i, c in enumerate(meta["shift_cases"]):
        words = [arr[f"se{i}_{j}"] for j in range(4)]
        assert eng.shifted_error_packed(*words, c["dx"], c["dy"]) == c["err"], c
        bm = [mtb.Bitmap(c["w"], c["h"], "packed", w) for w in words]
        assert mtb.shifted_error(*bm, mtb.ShiftOffset(c["dx"], c["dy"])) == c["err"]
        cells = [np.where(orc.unpack(w, c["w"]), 255, 0).astype(np.uint8) for w in words]
        assert eng.shifted_error_bytemap(*cells, c["dx"], c["dy"]) == c["err"], c
    wb = meta["word_boundary"]
    words = [arr[f"wb_{j}"] for j in range(4)]
    for c in wb["cases"]:
        assert eng.shifted_error_packed(*words, c["dx"], c["dy"]) == c["err"], c
    for i, c in enumerate(meta["count_cases"]):
        assert eng.count_ones_packed(arr[f"co{i}"]) == c["count"]


def test_shifted_error_symmetry_and_huge_offsets(mtb):
    rs = np.random.RandomState(17)
    for _ in range(6):
        w, h = int(rs.randint(5, 300)), int(rs.randint(5, 40))
        a, b = (mtb.Bitmap.from_bool(rs.rand(h, w) < 0.5) for _ in range(2))
        ea, eb = (mtb.Bitmap.from_bool(rs.rand(h, w) < 0.7) for _ in range(2))
        off = mtb.ShiftOffset(int(rs.randint(-70, 71)), int(rs.randint(-6, 7)))
        assert mtb.shifted_error(a, ea, b, eb, off) == mtb.shifted_error(b, eb, a, ea, -off)
        assert mtb.shifted_error(a, ea, b, eb, mtb.ShiftOffset(10 ** 7, 0)) == 0
        assert mtb.shifted_error(a, ea, b, eb, mtb.ShiftOffset(0, -h)) == 0


# ----------------------------------------------------------- golden: search --
def _check_result(res, want):
    assert list(res.offset) == want["offset"]
    assert res.total_tests == want["total_tests"]
    assert len(res.traces) == len(want["traces"])
    for t, w in zip(res.traces, want["traces"]):
        assert t.level == w["level"]
        assert list(t.chosen) == w["chosen"] and list(t.accumulated) == w["accumulated"]
        assert [[o.dx, o.dy, e] for o, e in t.candidates] == w["candidates"]


def test_find_offset_golden(mtb, golden):
    from paper_2007_06483_b200.instrumentation import SHIFTED_ERROR_EVALS, counters

    meta, arr = golden
    for c in meta["search_cases"]:
        rp = mtb.build_mtb_pyramid(mtb.build_pyramid(arr[f"srch_ref_{c['seed']}"], c["levels"]))
        tp = mtb.build_mtb_pyramid(mtb.build_pyramid(arr[f"srch_tgt_{c['seed']}"], c["levels"]))
        counters.reset()
        res = mtb.find_offset(rp, tp)
        assert counters.get(SHIFTED_ERROR_EVALS) == 9 * len(rp)
        _check_result(res, c["result"])
        off, err = mtb.brute_force_offset(rp[0], tp[0], 3)
        assert [off.dx, off.dy, err] == c["brute3"]
        # search_level with an explicit base reproduces the level-0 trace
        t0 = c["result"]["traces"][-1]
        base = mtb.ShiftOffset(t0["candidates"][4][0], t0["candidates"][4][1])
        chosen, cands = mtb.search_level(rp[0], tp[0], base)
        assert list(chosen) == t0["chosen"]
        assert [[o.dx, o.dy, e] for o, e in cands] == t0["candidates"]


def test_search_level_degenerate_ties_to_base(mtb):
    pair = mtb.make_mtb_pair(np.full((24, 24), 100, np.uint8))
    assert pair.exclusion.count_ones() == 0
    for base in (mtb.ShiftOffset(0, 0), mtb.ShiftOffset(6, -4)):
        chosen, cands = mtb.search_level(pair, pair, base)
        assert chosen == base and all(e == 0 for _, e in cands)


def test_align_stack_golden(mtb, golden):
    from paper_2007_06483_b200.instrumentation import FIND_OFFSET_CALLS, MTB_PYRAMID_BUILDS, PYRAMID_BUILDS, counters

    meta, _ = golden
    for c in meta["stack_cases"]:
        rng = np.random.default_rng(c["seed"])
        base = np.dstack([orc.smooth_gray(rng, c["w"], c["h"]) for _ in range(3)])
        gseed = int(rng.integers(2 ** 31))
        imgs, manifest = mtb.generate_stack(base, len(c["pairwise_in"]) + 1, pairwise=c["pairwise_in"], seed=gseed)
        assert [sha(im) for im in imgs] == c["input_sha"]        # device generator == reference generator
        counters.reset()
        aligned, record = mtb.align_stack(imgs)
        n = len(imgs)
        assert counters.get(PYRAMID_BUILDS) == n and counters.get(MTB_PYRAMID_BUILDS) == n
        assert counters.get(FIND_OFFSET_CALLS) == n - 1
        assert [list(x) for x in record.cumulative] == c["cumulative"]
        for r, want in zip(record.pairwise, c["pairwise"]):
            _check_result(r, want)
        assert aligned[0] is imgs[0]
        assert [sha(a) for a in aligned] == c["aligned_sha"]
        assert set(record.timings) == {"grayscale", "pyramid", "threshold", "search", "shift"}


def test_config1_golden_sweep(mtb, golden):
    meta, _ = golden
    rng = np.random.default_rng(0)
    base = np.dstack([orc.synthetic_gray(rng, 1024, 768) for _ in range(3)])
    assert sha(base) == meta["cfg1_base_sha"]
    for c in meta["cfg1"]:
        imgs, manifest = orc.generate_stack(base, 2, pairwise=c["pairwise_in"], seed=c["seed"], max_shift=63)
        assert [sha(im) for im in imgs] == c["input_sha"]
        aligned, record = mtb.align_stack(imgs)
        assert list(record.cumulative[1]) == c["offset"]
        _check_result(record.pairwise[0], c["result"])
        assert sha(aligned[1]) == c["aligned_sha"]
        assert mtb.get_exp_shift(imgs[0], imgs[1]) == tuple(c["offset"])


def test_degenerate_golden(mtb, golden):
    meta, _ = golden
    for c in meta["degenerate"]:
        img = np.full((96, 128, 3), c["value"], np.uint8)
        _, record = mtb.align_stack([img, img.copy()])
        assert list(record.cumulative[1]) == c["offset"]
        _check_result(record.pairwise[0], c["result"])


# ------------------------------------------------------ oracle at scale --
def _check_vs_oracle(res, want):
    assert tuple(res.offset) == tuple(want["offset"])
    for t, w in zip(res.traces, want["traces"]):
        assert t.level == w["level"] and tuple(t.chosen) == tuple(w["chosen"])
        assert [(o.dx, o.dy, e) for o, e in t.candidates] == [(o[0], o[1], e) for o, e in w["candidates"]]


def test_config1_random_sweep_vs_oracle(mtb, cuda):
    """32 more 1024x768 pairs (shifts up to 63) in ONE batched device search."""
    from paper_2007_06483_b200.engine import results_from_device

    rng = np.random.default_rng(5)
    base = np.dstack([orc.synthetic_gray(rng, 1024, 768) for _ in range(3)])
    imgs = []
    for s in range(32):
        pair, _ = orc.generate_stack(base, 2, seed=100 + s, max_shift=63)
        imgs.extend(pair)
    eng = mtb.MtbEngine(1024, 768, 6, 4)
    pyr = eng.preprocess(cuda.from_numpy(np.stack(imgs)).cuda())
    acc, errs = eng.search(pyr, [(2 * s, 2 * s + 1) for s in range(32)])
    got = results_from_device(acc, errs)
    for s in range(32):
        want = orc.align_pairs(imgs[2 * s:2 * s + 2], [(0, 1)])[0]
        _check_vs_oracle(got[s], want)


def test_24mp_pair_vs_oracle(mtb, cuda):
    """Config 2 size: one 6000x4000 pair, 6 levels — every trace, every L0 bitmap word."""
    rng = np.random.default_rng(1)
    base = np.dstack([orc.synthetic_gray(rng, 6000, 4000, cells=12) for _ in range(3)])
    imgs, man = orc.generate_stack(base, 2, seed=1, max_shift=63)
    eng = mtb.MtbEngine(6000, 4000, 6, 4)
    pyr = eng.preprocess(cuda.from_numpy(np.stack(imgs)).cuda())
    acc, errs = eng.search(pyr, [(0, 1)])
    from paper_2007_06483_b200.engine import results_from_device

    (res,) = results_from_device(acc, errs)
    want_pre = [orc.preprocess(im, 6, 4) for im in imgs]
    want = orc.find_offset(want_pre[0]["mtb"], want_pre[1]["mtb"])
    _check_vs_oracle(res, want)
    assert list(res.offset) == man["pairwise"][0]
    for i in range(2):
        for k in (0, 5):
            lv = want_pre[i]["mtb"][k]
            assert np.array_equal(eng.bitmap_words(pyr.mtb, i, k).cpu().numpy().view(np.uint64), orc.pack(lv["mtb"]))
            assert np.array_equal(eng.bitmap_words(pyr.excl, i, k).cpu().numpy().view(np.uint64),
                                  orc.pack(lv["excl"]))


def test_pivot_mode_vs_oracle(mtb):
    """Config 3 pairing (middle exposure as pivot) on a 7-exposure stack."""
    rng = np.random.default_rng(2)
    base = np.dstack([orc.synthetic_gray(rng, 800, 600) for _ in range(3)])
    gains = [2 ** ((k - 3) / 3) for k in range(7)]
    imgs, man = orc.generate_stack(base, 7, seed=2, max_shift=8, gains=gains, gammas=[1.0] * 7)
    aligned, record = mtb.align(imgs, mode="pivot")
    want_aligned, want_res, want_cum = orc.align_pivot(imgs, 3)
    assert [tuple(c) for c in record.cumulative] == [tuple(c) for c in want_cum]
    for r, w in zip(record.pairwise, want_res):
        _check_vs_oracle(r, w)
    assert aligned[3] is imgs[3]
    for a, w in zip(aligned, want_aligned):
        assert np.array_equal(a, w)
    # chain mode through `align` equals align_stack
    _, rec2 = mtb.align(imgs, mode="chain")
    _, rec3 = mtb.align_stack(imgs)
    assert rec2.cumulative == rec3.cumulative


def test_batch_equals_single(mtb, cuda):
    rng = np.random.default_rng(9)
    base = np.dstack([orc.synthetic_gray(rng, 640, 480) for _ in range(3)])
    imgs, _ = orc.generate_stack(base, 5, seed=9, max_shift=20)
    eng = mtb.MtbEngine(640, 480, 6, 4)
    pyr = eng.preprocess(cuda.from_numpy(np.stack(imgs)).cuda())
    pairs = [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0), (2, 2)]
    acc, errs = eng.search(pyr, pairs)
    for p, (r, t) in enumerate(pairs):
        a1, e1 = eng.search(pyr, [(r, t)])
        assert cuda.equal(acc[p], a1[0]) and cuda.equal(errs[p], e1[0])
    assert tuple(acc[5, 0].tolist()) == (0, 0)


# ---------------------------------------------------------- shifts / synth --
def test_shift_rgb_gray_vs_oracle(mtb):
    rs = np.random.RandomState(3)
    for _ in range(20):
        h, w = int(rs.randint(1, 40)), int(rs.randint(1, 40))
        img = rs.randint(0, 256, size=(h, w, 3), dtype=np.uint8)
        dx, dy = int(rs.randint(-w - 2, w + 3)), int(rs.randint(-h - 2, h + 3))
        fill = tuple(int(v) for v in rs.randint(0, 256, 3))
        assert np.array_equal(mtb.shift_rgb(img, mtb.ShiftOffset(dx, dy), fill), orc.shift_raster(img, dx, dy, fill))
        g = img[:, :, 0].copy()
        assert np.array_equal(mtb.shift_gray(g, mtb.ShiftOffset(dx, dy), 7), orc.shift_raster(g, dx, dy, 7))
    img = np.array([[[1, 2, 3], [4, 5, 6]]], dtype=np.uint8)
    assert mtb.shift_rgb(img, mtb.ShiftOffset(1, 0), fill=(9, 9, 9)).tolist() == [[[9, 9, 9], [1, 2, 3]]]
    big = np.arange(12, dtype=np.uint8).reshape(3, 4)
    assert (mtb.shift_gray(big, mtb.ShiftOffset(100, 0), fill=7) == 7).all()


def test_shift_rgb_vector_path_vs_oracle(mtb, cuda):
    """Rows of 3W % 16 == 0 take the 16-px vector kernel (PRMT byte funnels over
    aligned 16-B loads): every source misalignment, borders, fill, batches."""
    torch = cuda
    from paper_2007_06483_b200.image import shift_rgb_device
    rs = np.random.RandomState(11)
    for w, h in [(16, 5), (64, 9), (160, 33), (208, 17)]:
        imgs = rs.randint(0, 256, size=(6, h, w, 3), dtype=np.uint8)
        offs = [(int(d), int(rs.randint(-h, h + 1))) for d in rs.randint(-w - 3, w + 4, size=6)]
        offs[0] = (0, 0)
        offs[1] = (1, -1)
        fill = (5, 250, 17)
        out = shift_rgb_device(torch.from_numpy(imgs).cuda(), offs, fill).cpu().numpy()
        for i, (dx, dy) in enumerate(offs):
            assert np.array_equal(out[i], orc.shift_raster(imgs[i], dx, dy, fill)), (w, h, dx, dy)
    img = rs.randint(0, 256, size=(7, 48, 3), dtype=np.uint8)
    for dx in range(-20, 21):   # all 16 source byte alignments, both directions
        assert np.array_equal(mtb.shift_rgb(img, mtb.ShiftOffset(dx, 2), (1, 2, 3)),
                              orc.shift_raster(img, dx, 2, (1, 2, 3))), dx


def test_generate_stack_matches_reference_recipe(mtb):
    rng = np.random.default_rng(4)
    base = np.dstack([orc.smooth_gray(rng, 96, 80) for _ in range(3)])
    got, man = mtb.generate_stack(base, 4, seed=12, max_shift=9)
    want, wman = orc.generate_stack(base, 4, seed=12, max_shift=9)
    assert man["pairwise"] == wman["pairwise"] and man["cumulative"] == wman["cumulative"]
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
