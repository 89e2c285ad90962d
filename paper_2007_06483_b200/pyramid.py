"""2x box pyramids on the GPU (mirror of mtbalign.pyramid, pyramid.py:10-62).

down(x, y) = (2x2 block sum + 2) >> 2 with floor-halved dimensions; the
level count is min(requested, max_levels) where every level stays >= 16x16.
"""

from __future__ import annotations

from . import _dev, _lib
from .image import validate_gray
from .instrumentation import PYRAMID_BUILDS, counters

DEFAULT_LEVELS = 6
MIN_LEVEL_SIZE = 16


def _downsample_dev(src):
    torch = _dev.torch_mod()
    h, w = int(src.shape[0]), int(src.shape[1])
    out = torch.empty((h // 2, w // 2), dtype=torch.uint8, device="cuda")
    _lib.call("mtb_downsample_half", _dev.ptr(src), int(src.stride(0)), w, h, _dev.ptr(out), w // 2, _dev.stream())
    return out


def downsample_half(img):
    """Halve both dimensions by rounded 2x2 box averages (pyramid.py:17-32)."""
    validate_gray(img)
    h, w = _dev.shape_of(img)
    if h < 2 or w < 2:
        raise ValueError(f"a {w}x{h} image cannot be halved; at least 2x2 is required")
    return _dev.like_input(_downsample_dev(_dev.to_device(img)), img)


def max_levels(width: int, height: int) -> int:
    """Number of levels keeping every level at least 16x16 (pyramid.py:35-42)."""
    n = 0
    while width >= MIN_LEVEL_SIZE and height >= MIN_LEVEL_SIZE:
        n, width, height = n + 1, width // 2, height // 2
    return n


def build_pyramid(img, requested_levels: int = DEFAULT_LEVELS) -> list:
    """Halving pyramid; level 0 is the input object itself (pyramid.py:45-62)."""
    validate_gray(img)
    if requested_levels < 1:
        raise ValueError("requested_levels must be >= 1")
    h, w = _dev.shape_of(img)
    if w < MIN_LEVEL_SIZE or h < MIN_LEVEL_SIZE:
        raise ValueError(f"pyramids need images of at least 16x16; got {w}x{h}")
    counters.bump(PYRAMID_BUILDS)
    n = min(requested_levels, max_levels(w, h))
    levels = [img]
    cur = _dev.to_device(img) if n > 1 else None
    for _ in range(n - 1):
        cur = _downsample_dev(cur)
        levels.append(_dev.like_input(cur, img))
    return levels
