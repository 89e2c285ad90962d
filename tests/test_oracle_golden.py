"""Pin the CPU oracle to the reference: golden vectors made by the unmodified
reference (tests/golden/make_golden.py) and the reference tests' own
known answers.  CPU only."""

import hashlib

import numpy as np
import pytest

import mtb_oracle as orc


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---- known answers quoted from the reference test-suite ------------------
def test_known_answers():
    assert orc.gray(np.array([[[255, 0, 0]]], np.uint8))[0, 0] == 53           # test_image.py:25
    assert orc.gray(np.full((2, 3, 3), 255, np.uint8)).min() == 255            # test_image.py:21
    assert orc.downsample(np.array([[0, 0], [255, 255]], np.uint8))[0, 0] == 128  # test_pyramid.py:22
    p = orc.pyramid(np.zeros((1440, 2560), np.uint8), 6)                        # test_pyramid.py:66-70
    assert len(p) == 6 and p[-1].shape == (45, 80)
    p = orc.pyramid(np.zeros((64, 64), np.uint8), 6)                            # test_pyramid.py:72-76
    assert len(p) == 3 and p[-1].shape == (16, 16)
    assert orc.median(orc.histogram(np.array([[0, 1], [2, 3]], np.uint8))) == 1   # test_threshold.py:47
    assert orc.median(orc.histogram(np.array([[0, 255]] * 8, np.uint8))) == 0     # test_threshold.py:52
    ramp = np.repeat(np.arange(256, dtype=np.uint8), 4).reshape(32, 32)
    assert orc.median(orc.histogram(ramp)) == 127                               # test_threshold.py:94
    eb = orc.exclusion_mask(np.array([[100, 104, 105, 96, 95]], np.uint8), 100, 4)
    assert eb.tolist() == [[False, False, True, False, True]]                   # test_threshold.py:108
    assert not orc.exclusion_mask(np.array([[0]], np.uint8), 2, 4).any()        # no wrap near 0
    assert not orc.exclusion_mask(np.array([[255]], np.uint8), 253, 4).any()    # no wrap near 255
    with pytest.raises(ValueError):
        orc.median(np.zeros(256, np.int64))


def test_pack_padding_every_width():
    for w in range(1, 130):                                                     # test_bitmap.py:82-84
        words = orc.pack(np.ones((2, w), bool))
        assert words.shape == (2, (w + 63) // 64)
        assert int(np.bitwise_count(words).sum()) == 2 * w
        assert orc.unpack(words, w).all()


# ---- golden vectors from the reference -----------------------------------
def test_gray_golden(golden):
    _, arr = golden
    assert np.array_equal(orc.gray(arr["gray_in"]), arr["gray_out"])
    assert np.array_equal(orc.gray(arr["gray_solid_in"]), arr["gray_solid_out"])


def test_pyramid_threshold_golden(golden):
    meta, arr = golden
    for ci, case in enumerate(meta["pyramid_cases"]):
        img = arr[f"pyr{ci}_in"]
        levels = orc.pyramid(img, case["levels_requested"])
        assert len(levels) == case["n"]
        for k, lv in enumerate(levels):
            assert np.array_equal(lv, arr[f"pyr{ci}_l{k}"]), (ci, k)
            hist = orc.histogram(lv)
            assert np.array_equal(hist, arr[f"pyr{ci}_h{k}"])
            med = orc.median(hist)
            assert med == case["medians"][k]
            assert np.array_equal(orc.pack(orc.mtb_mask(lv, med)), arr[f"pyr{ci}_m{k}"])
            assert np.array_equal(orc.pack(orc.exclusion_mask(lv, med, case["tol"])), arr[f"pyr{ci}_e{k}"])


def test_shifted_error_golden(golden):
    meta, arr = golden
    for i, c in enumerate(meta["shift_cases"]):
        m = [orc.unpack(arr[f"se{i}_{j}"], c["w"]) for j in range(4)]
        assert orc.shifted_error(*m, c["dx"], c["dy"]) == c["err"], c
    wb = meta["word_boundary"]
    m = [orc.unpack(arr[f"wb_{j}"], wb["w"]) for j in range(4)]
    for c in wb["cases"]:
        assert orc.shifted_error(*m, c["dx"], c["dy"]) == c["err"], c


def _check_result(got, want):
    assert list(got["offset"]) == want["offset"]
    assert got["total_tests"] == want["total_tests"]
    for gt, wt in zip(got["traces"], want["traces"]):
        assert gt["level"] == wt["level"]
        assert list(gt["chosen"]) == wt["chosen"]
        assert [[o[0], o[1], e] for o, e in gt["candidates"]] == wt["candidates"]


def test_find_offset_golden(golden):
    meta, arr = golden
    for c in meta["search_cases"]:
        rp = orc.mtb_pyramid(orc.pyramid(arr[f"srch_ref_{c['seed']}"], c["levels"]), 4)
        tp = orc.mtb_pyramid(orc.pyramid(arr[f"srch_tgt_{c['seed']}"], c["levels"]), 4)
        _check_result(orc.find_offset(rp, tp), c["result"])
        (dx, dy), err = orc.brute_force(rp[0], tp[0], 3)
        assert [dx, dy, err] == c["brute3"]


def test_align_stack_golden(golden):
    meta, _ = golden
    for c in meta["stack_cases"]:
        rng = np.random.default_rng(c["seed"])
        base = np.dstack([orc.smooth_gray(rng, c["w"], c["h"]) for _ in range(3)])
        gseed = int(rng.integers(2 ** 31))
        assert gseed == c["gen_seed"]
        imgs, manifest = orc.generate_stack(base, len(c["pairwise_in"]) + 1, pairwise=c["pairwise_in"], seed=gseed)
        assert [sha(im) for im in imgs] == c["input_sha"]
        aligned, results, cum = orc.align_stack(imgs)
        assert [list(x) for x in cum] == c["cumulative"]
        for r, want in zip(results, c["pairwise"]):
            _check_result(r, want)
        assert [sha(a) for a in aligned] == c["aligned_sha"]


def test_config1_golden(golden):
    meta, _ = golden
    rng = np.random.default_rng(0)
    base = np.dstack([orc.synthetic_gray(rng, 1024, 768) for _ in range(3)])
    assert sha(base) == meta["cfg1_base_sha"]
    for c in meta["cfg1"][:3]:  # the full sweep runs in the GPU parity suite
        imgs, manifest = orc.generate_stack(base, 2, pairwise=c["pairwise_in"], seed=c["seed"], max_shift=63)
        assert [sha(im) for im in imgs] == c["input_sha"]
        assert manifest["pairwise"] == c["manifest_pairwise"]
        aligned, results, cum = orc.align_stack(imgs)
        assert list(cum[1]) == c["offset"]
        _check_result(results[0], c["result"])
        assert sha(aligned[1]) == c["aligned_sha"]


def test_degenerate_golden(golden):
    meta, _ = golden
    for c in meta["degenerate"]:
        img = np.full((96, 128, 3), c["value"], np.uint8)
        _, results, cum = orc.align_stack([img, img.copy()])
        assert list(cum[1]) == c["offset"] == [0, 0]
        _check_result(results[0], c["result"])
