"""GPU parity at the BASELINE configs' stated sizes, the reference's
acceptance criteria 3, 4 and 6 on the GPU path, and the round-2 host APIs.

Bit-exact (tolerance 0: integer path) against the CPU oracle
(oracle/mtb_oracle.py, pinned to the reference by tests/test_oracle_golden.py):
  * config 4 shape (4000x3000) through the fused pipeline, 2 images per launch;
  * config 3 (a 7-exposure 6000x4000 stack aligned to its middle exposure,
    SURVEY 8(d) recipe) through `align(mode="pivot")` = the fused pipeline;
  * a 10-level pyramid (8192x8192, levels 7-9 from the staged tail passes);
  * config 5's size (40000x25000, RGB batch > 2^31 bytes: 64-bit offsets)
    staged vs the row-sharded loopback (GPU vs GPU: the oracle needs ~30 GB);
  * a pivot plan with more pairs than one fused launch carries (120 frames
    aligned to the last one).
Acceptance criteria (/root/reference/pkg/tests/test_acceptance.py):
  3 (:110-136) pyramid search == brute force at radius 8, 200 cases;
  4 (:139-172) packed == bytemap shifted_error, 1000 cases over all 64 width
    residues, and end-to-end layout parity;
  6 (:209-226) MTB invariance under monotone tone curves.
"""

import time

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


def _check_pre(eng, pyr, imgs, levels, tol=4):
    """Medians and every packed map of every image equal the oracle's."""
    med = pyr.medians.cpu().numpy()
    pre = []
    for i, im in enumerate(imgs):
        p = orc.preprocess(im, levels, tol)
        pre.append(p)
        assert [lv["median"] for lv in p["mtb"]] == med[i].tolist(), i
        for k in range(eng.n):
            assert np.array_equal(eng.bitmap_words(pyr.mtb, i, k).cpu().numpy().view(np.uint64),
                                  orc.pack(p["mtb"][k]["mtb"])), (i, k)
            assert np.array_equal(eng.bitmap_words(pyr.excl, i, k).cpu().numpy().view(np.uint64),
                                  orc.pack(p["mtb"][k]["excl"])), (i, k)
    return pre


def _check_traces(acc, errs, pre, pairs):
    acc_h, errs_h = acc.cpu().numpy(), errs.cpu().numpy()
    for q, (r, t) in enumerate(pairs):
        want = orc.find_offset(pre[r]["mtb"], pre[t]["mtb"])
        assert tuple(acc_h[q, 0]) == tuple(want["offset"]), (q, acc_h[q, 0], want["offset"])
        for tr in want["traces"]:
            assert [e for _, e in tr["candidates"]] == errs_h[q, tr["level"]].tolist(), (q, tr["level"])
            assert tuple(acc_h[q, tr["level"]]) == tuple(tr["chosen"]), (q, tr["level"])


def test_config4_fused_vs_oracle(mtb, cuda):
    """4000 x 3000 (config 4's pair size), 2 pairs = 2 launches of 2 images."""
    from paper_2007_06483_b200.synth import generate_stack, synthetic_rgb_device

    w, h = 4000, 3000
    eng = mtb.MtbEngine(w, h, 6, 4)
    # the API dispatches 12 MP to the staged kernels (equal speed there); the
    # fused pipeline is tested directly at this size
    assert eng.fused_supported and not mtb.pipeline.use_fused(eng, 4)
    assert eng.fused_launches(4, [(0, 1), (2, 3)]) > 2
    imgs = []
    for s in range(2):
        st, _ = generate_stack(synthetic_rgb_device(40 + s, w, h), 2, seed=40 + s, max_shift=63)
        imgs += st
    batch = cuda.stack(imgs).contiguous()
    pyr, acc, errs = eng.align_fused(batch, [(0, 1), (2, 3)])
    host = [im.cpu().numpy() for im in imgs]
    pre = _check_pre(eng, pyr, host, 6)
    _check_traces(acc, errs, pre, [(0, 1), (2, 3)])


def test_config4_staged_vs_oracle(mtb, cuda):
    """4000 x 3000 through the staged kernels the API dispatches 12 MP to:
    rows of 63 u64 words (the search stages 8-byte chunks), offsets up to 63
    px (halo chunks past both row ends), medians, maps and every trace."""
    from paper_2007_06483_b200.synth import generate_stack, synthetic_rgb_device

    w, h = 4000, 3000
    eng = mtb.MtbEngine(w, h, 6, 4)
    assert not mtb.pipeline.use_fused(eng, 4) and (int(eng.geom[0, 4]) * 2) % 4 == 2
    imgs = []
    for s in range(2):
        st, _ = generate_stack(synthetic_rgb_device(50 + s, w, h), 2, seed=50 + s, max_shift=63)
        imgs += st
    batch = cuda.stack(imgs).contiguous()
    pyr = eng.preprocess(batch)
    acc, errs = eng.search(pyr, [(0, 1), (2, 3)])
    host = [im.cpu().numpy() for im in imgs]
    pre = _check_pre(eng, pyr, host, 6)
    _check_traces(acc, errs, pre, [(0, 1), (2, 3)])


def test_config3_pivot_stack_fused_vs_oracle(mtb, cuda):
    """7 x 6000 x 4000 aligned to exposure 3 (SURVEY 8(d) config 3 recipe) via
    align(mode="pivot") (staged for one stack) and the fused pipeline:
    offsets, every trace and the aligned outputs."""
    from paper_2007_06483_b200.synth import generate_stack, synthetic_rgb_device

    w, h = 6000, 4000
    base = synthetic_rgb_device(2, w, h)
    imgs, man = generate_stack(base, 7, seed=2, max_shift=20, gains=[2 ** ((k - 3) / 3) for k in range(7)],
                               gammas=[1.0] * 7)
    eng = mtb.pipeline.engine_for(w, h, 6, 4)
    assert not mtb.pipeline.use_fused(eng, 7)   # one 7-stack: staged is the faster call
    aligned, rec = mtb.align(imgs, mode="pivot")
    host = [im.cpu().numpy() for im in imgs]
    pre = [orc.preprocess(im, 6, 4) for im in host]
    # the fused pipeline on the same stack (what config 3's batches of 16 stacks use)
    pivot = [(3, i) for i in range(7) if i != 3]
    _, facc, ferrs = eng.align_fused(cuda.stack(imgs).contiguous(), pivot)
    _check_traces(facc, ferrs, pre, pivot)
    for (ref, tgt), res in zip([(3, i) for i in range(7) if i != 3], rec.pairwise):
        want = orc.find_offset(pre[ref]["mtb"], pre[tgt]["mtb"])
        assert tuple(res.offset) == tuple(want["offset"]), (tgt, res.offset, want["offset"])
        for t, wt in zip(res.traces, want["traces"]):
            assert [e for _, e in t.candidates] == [e for _, e in wt["candidates"]], (tgt, t.level)
        assert tuple(rec.cumulative[tgt]) == tuple(want["offset"])
        out = aligned[tgt].cpu().numpy()
        assert np.array_equal(out, orc.shift_raster(host[tgt], *want["offset"], fill=(0, 0, 0))), tgt
    assert aligned[3] is imgs[3]


def test_ten_level_pyramid_vs_oracle(mtb, cuda):
    """8192 x 8192 with levels=10: medians and maps of all 10 levels (7-9 from
    the staged tail passes) and the 10-level search traces."""
    from paper_2007_06483_b200.image import shift_rgb_device
    from paper_2007_06483_b200.synth import apply_lut_device, synthetic_rgb_device, tone_lut

    w = h = 8192
    eng = mtb.MtbEngine(w, h, 10, 4)
    assert eng.n == 10
    base = synthetic_rgb_device(9, w, h)
    moved = shift_rgb_device(base.unsqueeze(0), [(-150, 90)])[0]
    batch = cuda.empty((2, h, w, 3), dtype=cuda.uint8, device="cuda")
    apply_lut_device(base, tone_lut(1.2, 1.1), out=batch[0])
    apply_lut_device(moved, tone_lut(0.8, 0.9), out=batch[1])
    pyr = eng.preprocess(batch)
    acc, errs = eng.search(pyr, [(0, 1)])
    host = [batch[i].cpu().numpy() for i in range(2)]
    pre = _check_pre(eng, pyr, host, 10)
    _check_traces(acc, errs, pre, [(0, 1)])


def test_gigapixel_staged_equals_row_sharded(mtb, cuda):
    """40000 x 25000 (config 5's size, 10 levels; the 2-image batch is 6 GB, so
    every byte offset past 2^31 is exercised) on one GPU: the staged engine and
    the 8-shard row-sharded loopback agree bit for bit."""
    from paper_2007_06483_b200.engine import results_from_device
    from paper_2007_06483_b200.image import shift_rgb_device
    from paper_2007_06483_b200.sharded import align_pair_loopback
    from paper_2007_06483_b200.synth import synthetic_rgb_device

    w, h = 40000, 25000
    batch = cuda.empty((2, h, w, 3), dtype=cuda.uint8, device="cuda")
    batch[0].copy_(synthetic_rgb_device(5, w, h))
    shift_rgb_device(batch[0].unsqueeze(0), [(-301, 177)], out=batch[1].unsqueeze(0))
    eng = mtb.MtbEngine(w, h, 10, 4)
    assert eng.n == 10
    pyr = eng.preprocess(batch)
    acc, errs = eng.search(pyr, [(0, 1)])
    (staged,) = results_from_device(acc, errs)
    del pyr
    cuda.cuda.empty_cache()
    sharded = align_pair_loopback(batch[0], batch[1], 8, levels=10)
    assert tuple(staged.offset) == tuple(sharded.offset)
    for a, b in zip(staged.traces, sharded.traces):
        assert a.level == b.level and a.chosen == b.chosen
        assert [e for _, e in a.candidates] == [e for _, e in b.candidates], a.level


@pytest.mark.parametrize("n_img", [120, 230])
def test_fused_plan_more_pairs_than_one_launch(mtb, cuda, n_img):
    """Every frame aligned to the LAST one: all n-1 pairs become ready in the
    same launch (> 96 items); the plan spreads them over later launches before
    enqueueing anything.  Equal to the staged search, bit for bit."""
    from paper_2007_06483_b200.synth import generate_stack, synthetic_rgb_device

    w, h = 256, 192
    steps = [(1 + (i % 3), 1) if i % 2 == 0 else (-(1 + (i % 3)), -1) for i in range(n_img - 1)]   # bounded drift
    imgs, _ = generate_stack(synthetic_rgb_device(3, w, h), n_img, pairwise=steps, seed=3)
    batch = cuda.stack(imgs).contiguous()
    pairs = [(n_img - 1, i) for i in range(n_img - 1)]
    eng = mtb.MtbEngine(w, h, 6, 4)
    pyr_f, acc_f, errs_f = eng.align_fused(batch, pairs)
    pyr_s = eng.preprocess(batch)
    acc_s, errs_s = eng.search(pyr_s, pairs)
    assert cuda.equal(acc_f, acc_s) and cuda.equal(errs_f, errs_s)
    assert cuda.equal(pyr_f.medians, pyr_s.medians)


def test_align_stacks_equals_per_stack_align(mtb, cuda):
    """align_stacks (one device batch) == align on each stack: staged (640x480)
    and fused (2048x2048 = 4.2 MP) sizes, chain and pivot pairing."""
    from paper_2007_06483_b200.synth import generate_stack, synthetic_rgb_device

    for (w, h), mode in (((640, 480), "chain"), ((2048, 2048), "pivot")):
        stacks = [generate_stack(synthetic_rgb_device(60 + s, w, h), 3 + s, seed=60 + s, max_shift=12)[0]
                  for s in range(3)]
        batched = mtb.align_stacks(stacks, mode=mode)
        assert len(batched) == 3
        for st, (aligned, rec) in zip(stacks, batched):
            ref_aligned, ref_rec = mtb.align(st, mode=mode)
            assert rec.cumulative == ref_rec.cumulative
            assert [r.offset for r in rec.pairwise] == [r.offset for r in ref_rec.pairwise]
            assert all(cuda.equal(a, b) for a, b in zip(aligned, ref_aligned))


def test_stage_timings_from_events(mtb, cuda):
    """STAGES come from CUDA events (pipeline.py:74-112): all five, non-negative,
    summing to the call's wall time (within host jitter); 0 threshold time in
    fused mode, where it overlaps the pipeline."""
    from paper_2007_06483_b200.pipeline import STAGES
    from paper_2007_06483_b200.synth import generate_stack, synthetic_rgb_device

    for w, h in ((800, 600), (2048, 2048)):
        imgs = [im.cpu().numpy() for im in generate_stack(synthetic_rgb_device(7, w, h), 3, seed=7)[0]]
        mtb.align_stack(imgs)
        t0 = time.perf_counter()
        _, rec = mtb.align_stack(imgs)
        wall = (time.perf_counter() - t0) * 1000.0
        assert tuple(rec.timings) == STAGES
        assert all(v >= 0.0 for v in rec.timings.values())
        total = sum(rec.timings.values())
        assert total <= wall * 1.05 + 1.0 and total >= wall * 0.5, (total, wall)
        if mtb.pipeline.use_fused(mtb.pipeline.engine_for(w, h, 6, 4), len(imgs)):
            assert rec.timings["threshold"] == pytest.approx(0.0, abs=0.05)


def test_second_device_when_present(mtb, cuda):
    """Per-device SM count and shared-memory opt-in: the fused and staged
    paths run on cuda:1 and agree with cuda:0."""
    if cuda.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    from paper_2007_06483_b200.synth import generate_stack, synthetic_rgb_device

    results = []
    for dev in (0, 1):
        with cuda.cuda.device(dev):
            imgs = generate_stack(synthetic_rgb_device(8, 2400, 1800), 2, seed=8)[0]
            results.append((tuple(mtb.get_exp_shift(imgs[0], imgs[1])),
                            [tuple(c) for c in mtb.align_stack(imgs)[1].cumulative]))
    assert results[0] == results[1]


# ---- acceptance criteria on the GPU path -----------------------------------
def test_acceptance_3_pyramid_equals_brute_force(mtb, cuda):
    """test_acceptance.py:110-136: 200 random 64..128 px images shifted by up to
    7 px (fill = median), 3 levels; on every non-degenerate case the pyramid
    search equals the radius-8 brute force — both on the device."""
    rng = np.random.default_rng(1234)
    usable = agree = 0
    for _ in range(200):
        w, h = int(rng.integers(64, 129)), int(rng.integers(64, 129))
        gray = orc.smooth_gray(rng, w, h)
        shift = mtb.ShiftOffset(int(rng.integers(-7, 8)), int(rng.integers(-7, 8)))
        med = mtb.median_from_histogram(mtb.histogram(gray))
        moved = mtb.shift_gray(gray, shift, fill=med)
        ref = mtb.build_mtb_pyramid(mtb.build_pyramid(gray, 3))
        tgt = mtb.build_mtb_pyramid(mtb.build_pyramid(moved, 3))
        if any(p.exclusion.count_ones() < 0.05 * p.exclusion.width * p.exclusion.height for p in ref + tgt):
            continue
        usable += 1
        got = mtb.find_offset(ref, tgt).offset
        brute, _ = mtb.brute_force_offset(ref[0], tgt[0], 8)
        agree += got == brute
    assert usable > 100 and agree == usable, (agree, usable)


def test_acceptance_4_layout_parity(mtb, cuda):
    """test_acceptance.py:139-172: packed and bytemap shifted_error agree (and
    equal the oracle) on 1000 random cases sweeping every width residue mod 64
    with offsets beyond the raster; 12 stacks align identically in both layouts."""
    rng = np.random.default_rng(4444)
    residues = set()
    for i in range(1000):
        w = 1 + (i % 128)
        h = int(rng.integers(1, 25))
        residues.add(w % 64)
        masks = [rng.random((h, w)) < rng.random() for _ in range(4)]
        dx, dy = int(rng.integers(-w - 65, w + 66)), int(rng.integers(-h - 2, h + 3))
        errs = []
        for layout in mtb.LAYOUTS:
            maps = [mtb.Bitmap.from_bool(m, layout) for m in masks]
            errs.append(mtb.shifted_error(*maps, mtb.ShiftOffset(dx, dy)))
        want = orc.shifted_error(*[m.astype(np.uint8) for m in masks], dx, dy)
        assert errs[0] == errs[1] == want, (i, w, h, dx, dy, errs, want)
    assert residues == set(range(64))
    for trial in range(12):
        base = np.dstack([orc.smooth_gray(rng, 160 + trial, 140) for _ in range(3)])
        imgs, _ = orc.generate_stack(base, 3, seed=trial, max_shift=10)
        offs = [[tuple(o) for o in mtb.align_stack(imgs, layout=lay)[1].cumulative] for lay in (mtb.PACKED, mtb.BYTEMAP)]
        assert offs[0] == offs[1], trial


def _monotone_curve(rng, occupied):
    """Tone curve strictly increasing on the occupied values (the reference
    conftest's random_monotone_curve recipe, test infrastructure)."""
    vals = np.flatnonzero(occupied)
    targets = np.sort(rng.choice(256, size=vals.size, replace=False))
    curve = np.zeros(256, dtype=np.uint8)
    pv, pt = 0, targets[0]
    for v, t in zip(vals, targets):
        curve[pv:v + 1] = np.linspace(pt, t, v - pv + 1).astype(np.uint8)
        curve[v] = t
        pv, pt = v, t
    curve[pv:] = pt
    return curve


def test_acceptance_6_mtb_exposure_invariance(mtb, cuda):
    """test_acceptance.py:209-226: the device MTB of an image equals the MTB of
    any strictly monotone re-toning of it (100 random cases)."""
    rng = np.random.default_rng(66)
    for _ in range(100):
        w, h = int(rng.integers(16, 64)), int(rng.integers(16, 64))
        img = rng.integers(0, 256, size=(h, w)).astype(np.uint8)
        occ = np.zeros(256, dtype=bool)
        occ[np.unique(img)] = True
        curve = _monotone_curve(rng, occ)
        before = mtb.make_mtb_pair(img).mtb.to_bool()
        after = mtb.make_mtb_pair(curve[img]).mtb.to_bool()
        assert np.array_equal(before, after)


def test_concurrent_fused_calls_on_two_streams(mtb, cuda):
    """Two host threads run align_fused on the SAME engine on different
    streams at once: per-call scratch (gray ring, sync words) keeps them
    independent; results equal the serial ones."""
    import threading

    from paper_2007_06483_b200.synth import generate_stack, synthetic_rgb_device

    w, h = 2048, 1536
    eng = mtb.MtbEngine(w, h, 6, 4)
    batches = [cuda.stack(generate_stack(synthetic_rgb_device(30 + i, w, h), 6, seed=30 + i, max_shift=20)[0])
               for i in range(2)]
    pairs = [(0, 1), (1, 2), (3, 4), (4, 5), (0, 5)]
    serial = [eng.align_fused(b, pairs)[1].clone() for b in batches]
    out = [None, None]

    def run(i):
        s = cuda.cuda.Stream()
        with cuda.cuda.stream(s):
            for _ in range(5):
                _, acc, _ = eng.align_fused(batches[i], pairs)
            out[i] = acc.clone()
        s.synchronize()

    ts = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in range(2):
        assert cuda.equal(out[i], serial[i])


def test_random_geometry_sweep_vs_oracle(mtb, cuda):
    """24 seeded random cases through the public API (align_stack /
    align(mode="pivot")): widths 16..2600 (multiples of 16 take the fused
    path at >= 4 MP-equivalent batches only when large, else staged), odd and
    even heights, 1..6 levels, tolerances 0..200; every pairwise offset, every
    trace's 9 counts and the aligned outputs equal the oracle's."""
    rng = np.random.default_rng(20261017)
    for case in range(24):
        w = int(rng.integers(16, 2600))
        if case % 3 == 0:
            w = max(16, w - w % 16)                     # TMA-friendly width
        h = int(rng.integers(16, 1700))
        levels = int(rng.integers(1, 7))
        tol = int(rng.choice([0, 1, 4, 7, 31, 127, 128, 200]))
        count = int(rng.integers(2, 5))
        base = np.dstack([orc.smooth_gray(rng, w, h, cells=6) for _ in range(3)])
        imgs, _ = orc.generate_stack(base, count, seed=case, max_shift=min(12, max(1, min(w, h) // 8)))
        mode = "pivot" if case % 2 else "chain"
        aligned, rec = mtb.align(imgs, levels=levels, tol=tol, mode=mode)
        if mode == "chain":
            want_al, want_res, want_cum = orc.align_stack(imgs, levels, tol)
        else:
            want_al, want_res, want_cum = orc.align_pivot(imgs, count // 2, levels, tol)
        assert [tuple(c) for c in rec.cumulative] == [tuple(c) for c in want_cum], (case, w, h, levels, tol)
        for res, want in zip(rec.pairwise, want_res):
            for t, wt in zip(res.traces, want["traces"]):
                assert [e for _, e in t.candidates] == [e for _, e in wt["candidates"]], (case, t.level)
        for a, b in zip(aligned, want_al):
            assert np.array_equal(np.asarray(a), b), case
