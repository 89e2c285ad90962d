"""Host-side logic of the drop-in API that needs no GPU: engine registry,
validation errors (raised before any device work), dataclasses, counters,
trace reconstruction."""

import numpy as np
import pytest
import torch

import paper_2007_06483_b200 as mtb
from paper_2007_06483_b200 import kernels
from paper_2007_06483_b200.engine import results_from_device
from paper_2007_06483_b200.pipeline import STAGES
from paper_2007_06483_b200.pyramid import max_levels
from paper_2007_06483_b200.search import NEIGHBORHOOD


def test_public_names_cover_reference_hot_path():
    ref_all = {"AlignmentResult", "BYTEMAP", "Bitmap", "LAYOUTS", "LevelTrace", "MtbPair", "PACKED", "ShiftOffset",
               "StackAlignment", "align_stack", "brute_force_offset", "build_mtb_pyramid", "build_pyramid",
               "downsample_half", "find_offset", "generate_stack", "histogram", "make_exclusion", "make_mtb",
               "make_mtb_pair", "measure_alignment", "median_from_histogram", "search_level", "shift_gray",
               "shift_rgb", "shifted_error", "to_grayscale"}
    assert ref_all <= set(mtb.__all__)
    assert {"align", "get_exp_shift"} <= set(mtb.__all__)
    for name in mtb.__all__:
        assert hasattr(mtb, name)


def test_engine_registry_has_no_cpu_fallback():
    assert kernels.use("auto") == "cuda"
    assert kernels.use("native") == "cuda"
    assert kernels.engine_name() == "cuda"
    with pytest.raises(RuntimeError):
        kernels.use("python")
    with pytest.raises(ValueError):
        kernels.use("gpu")
    assert kernels.engine_name() == "cuda"


def test_shift_offset_algebra():
    a = mtb.ShiftOffset(3, -2)
    assert -a == (-3, 2)
    assert a + (1, 1) == (4, -1)
    assert a.scaled(2) == (6, -4)


def test_neighborhood_scan_order():
    assert NEIGHBORHOOD == ((-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 0), (0, 1), (1, -1), (1, 0), (1, 1))


def test_max_levels():
    assert max_levels(2560, 1440) == 7 and max_levels(64, 64) == 3 and max_levels(15, 99) == 0


@pytest.mark.parametrize("bad", [np.zeros((4, 4), np.uint8), np.zeros((4, 4, 3), np.float32), "x",
                                 np.zeros((0, 4, 3), np.uint8)])
def test_rgb_validation_before_device(bad):
    with pytest.raises(ValueError):
        mtb.to_grayscale(bad)


def test_gray_validation_before_device():
    with pytest.raises(ValueError):
        mtb.build_pyramid(np.zeros((15, 40), np.uint8), 2)
    with pytest.raises(ValueError):
        mtb.build_pyramid(np.zeros((32, 32), np.uint8), 0)
    with pytest.raises(ValueError):
        mtb.downsample_half(np.zeros((1, 5), np.uint8))
    with pytest.raises(ValueError):
        mtb.histogram(np.zeros((3, 3, 3), np.uint8))


def test_stack_validation_before_device():
    a = np.zeros((32, 32, 3), np.uint8)
    with pytest.raises(ValueError):
        mtb.align_stack([a])
    with pytest.raises(ValueError):
        mtb.align_stack([a, np.zeros((32, 33, 3), np.uint8)])
    with pytest.raises(ValueError):
        mtb.align_stack([np.zeros((8, 8, 3), np.uint8)] * 2)
    with pytest.raises(ValueError):
        mtb.align([a, a], mode="bogus")
    with pytest.raises(ValueError):
        mtb.measure_alignment([a, a], repetitions=0)


def test_trace_reconstruction_from_device_buffers():
    # Two levels; level 1 chose (1, 0) around base (0, 0); level 0 chose (3, -1) around (2, 0).
    acc = torch.tensor([[[3, -1], [1, 0]]], dtype=torch.int32)
    errs = torch.arange(18, dtype=torch.int64).reshape(1, 2, 9)
    (res,) = results_from_device(acc, errs)
    assert res.offset == (3, -1) and res.total_tests == 18
    t1, t0 = res.traces
    assert t1.level == 1 and t0.level == 0
    assert [tuple(o) for o, _ in t1.candidates] == [(ddx, ddy) for ddy, ddx in NEIGHBORHOOD]
    assert [tuple(o) for o, _ in t0.candidates] == [(2 + ddx, ddy) for ddy, ddx in NEIGHBORHOOD]
    assert [e for _, e in t0.candidates] == list(range(9))
    assert t0.chosen == t0.accumulated == (3, -1)


def test_stage_names():
    assert STAGES == ("grayscale", "pyramid", "threshold", "search", "shift")


def test_tone_lut_matches_oracle():
    import mtb_oracle as orc
    from paper_2007_06483_b200.synth import draw_manifest, tone_lut

    for gain, gamma in [(0.5, 0.7), (2.0, 1.4), (1.3, 1.0)]:
        assert np.array_equal(tone_lut(gain, gamma), orc.tone_lut(gain, gamma))
    pw, cum, gains, gammas = draw_manifest(4, seed=9, max_shift=7)
    _, man = orc.generate_stack(np.zeros((64, 64, 3), np.uint8), 4, seed=9, max_shift=7)
    assert [list(o) for o in pw] == man["pairwise"] and gains == man["gains"] and gammas == man["gammas"]
