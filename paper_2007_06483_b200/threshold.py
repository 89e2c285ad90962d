"""Histograms, medians and MTB / exclusion bitmaps on the GPU.

Mirrors mtbalign.threshold (pkg/src/mtbalign/threshold.py:22-88).  The MTB
marks pixels strictly above the level's median; the exclusion bitmap marks
pixels farther than `tol` from it (set = reliable, the reference's
polarity, threshold.py:7-9).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .bitmap import PACKED, Bitmap, _check_layout, words_per_row
from .image import validate_gray
from .instrumentation import MTB_PYRAMID_BUILDS, counters

DEFAULT_NOISE_TOLERANCE = 4


def _hist_dev(src):
    torch = _dev.torch_mod()
    h, w = int(src.shape[0]), int(src.shape[1])
    out = torch.empty(256, dtype=torch.int64, device="cuda")
    _lib.call("mtb_histogram", _dev.ptr(src), int(src.stride(0)), w, h, _dev.ptr(out), _dev.stream())
    return out


def histogram(img):
    """256-bin histogram, int64 bins summing to H*W (threshold.py:25-28)."""
    validate_gray(img)
    return _dev.like_input(_hist_dev(_dev.to_device(img)), img)


def _median_dev(hist_dev):
    """Device lower median of a (.., 256) int64 tensor; int32 tensor out (-1 = empty)."""
    torch = _dev.torch_mod()
    flat = hist_dev.reshape(-1, 256).contiguous()
    med = torch.empty(flat.shape[0], dtype=torch.int32, device="cuda")
    _lib.call("mtb_median_from_histogram", _dev.ptr(flat), int(flat.shape[0]), _dev.ptr(med), _dev.stream())
    return med


def median_from_histogram(hist) -> int:
    """Smallest value whose cumulative count reaches ceil(total/2) (threshold.py:31-39)."""
    torch = _dev.torch_mod()
    h = _dev.to_device(np.asarray(hist, dtype=np.int64) if isinstance(hist, (np.ndarray, list, tuple))
                       else hist, torch.int64)
    if h.numel() != 256:
        raise ValueError(f"expected a 256-bin histogram, got {h.numel()} bins")
    med = int(_median_dev(h).item())
    if med < 0:
        raise ValueError("the median of an empty histogram is undefined")
    return med


def _threshold_dev(src, median: int, tol: int, want_mtb: bool, want_excl: bool):
    torch = _dev.torch_mod()
    h, w = int(src.shape[0]), int(src.shape[1])
    shape = (h, words_per_row(w))
    mtb = torch.empty(shape, dtype=torch.int64, device="cuda") if want_mtb else None
    excl = torch.empty(shape, dtype=torch.int64, device="cuda") if want_excl else None
    _lib.call("mtb_threshold_pack", _dev.ptr(src), int(src.stride(0)), w, h, int(median), int(tol),
              _dev.ptr(mtb) if mtb is not None else None, _dev.ptr(excl) if excl is not None else None,
              _dev.stream())
    return mtb, excl


def make_mtb(img, median: int, layout: str = PACKED) -> Bitmap:
    """1 where pixel > median (threshold.py:42-45)."""
    validate_gray(img)
    _check_layout(layout)
    src = _dev.to_device(img)
    mtb, _ = _threshold_dev(src, median, 0, True, False)
    return Bitmap(int(src.shape[1]), int(src.shape[0]), layout, mtb)


def make_exclusion(img, median: int, tol: int = DEFAULT_NOISE_TOLERANCE, layout: str = PACKED) -> Bitmap:
    """1 where |pixel - median| > tol, in widened integers (threshold.py:48-56)."""
    validate_gray(img)
    _check_layout(layout)
    src = _dev.to_device(img)
    _, excl = _threshold_dev(src, median, tol, False, True)
    return Bitmap(int(src.shape[1]), int(src.shape[0]), layout, excl)


@dataclass(frozen=True)
class MtbPair:
    """MTB and exclusion bitmap of one image at one level (threshold.py:59-66)."""

    mtb: Bitmap
    exclusion: Bitmap
    median: int
    noise_tolerance: int


def make_mtb_pair(img, tol: int = DEFAULT_NOISE_TOLERANCE, layout: str = PACKED) -> MtbPair:
    """Histogram -> median -> both bitmaps in one device pass (threshold.py:69-77)."""
    validate_gray(img)
    _check_layout(layout)
    src = _dev.to_device(img)
    med = int(_median_dev(_hist_dev(src)).item())
    mtb, excl = _threshold_dev(src, med, tol, True, True)
    w, h = int(src.shape[1]), int(src.shape[0])
    return MtbPair(mtb=Bitmap(w, h, layout, mtb), exclusion=Bitmap(w, h, layout, excl), median=med,
                   noise_tolerance=tol)


def build_mtb_pyramid(levels: list, tol: int = DEFAULT_NOISE_TOLERANCE, layout: str = PACKED) -> list:
    """One MtbPair per level, each from the level's own median (threshold.py:80-88)."""
    counters.bump(MTB_PYRAMID_BUILDS)
    return [make_mtb_pair(level, tol, layout) for level in levels]
