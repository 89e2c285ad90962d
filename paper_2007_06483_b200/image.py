"""Raster validation, grayscale conversion and whole-pixel shifts on the GPU.

Mirrors mtbalign.image (pkg/src/mtbalign/image.py).  Images are uint8
numpy arrays or torch CUDA tensors: RGB (H, W, 3) interleaved, gray (H, W).
A ShiftOffset (dx, dy) moves content right by dx and down by dy.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np

from . import _dev, _lib

# image.py:17-19 — integer BT.601-style weights summing to 256.
GRAY_WEIGHT_R = 54
GRAY_WEIGHT_G = 183
GRAY_WEIGHT_B = 19


class ShiftOffset(NamedTuple):
    """Signed whole-pixel translation (image.py:22-35): +dx right, +dy down."""

    dx: int
    dy: int

    def __neg__(self) -> "ShiftOffset":
        return ShiftOffset(-self.dx, -self.dy)

    def __add__(self, other) -> "ShiftOffset":
        return ShiftOffset(self.dx + other[0], self.dy + other[1])

    def scaled(self, factor: int) -> "ShiftOffset":
        return ShiftOffset(self.dx * factor, self.dy * factor)


def validate_rgb(img):
    """(H, W, 3) uint8 with H, W >= 1, else ValueError (image.py:38-45)."""
    shape = _dev.shape_of(img)
    if shape is None or len(shape) != 3 or shape[2] != 3 or not (
            isinstance(img, np.ndarray) or _dev.is_tensor(img)):
        raise ValueError(f"RGB image must have shape (H, W, 3); got {shape}")
    if not _dev.is_u8(img):
        raise ValueError(f"RGB samples must be uint8; got {_dev.dtype_name(img)}")
    if shape[0] < 1 or shape[1] < 1:
        raise ValueError("image must be at least 1x1")
    return img


def validate_gray(img):
    """(H, W) uint8 with H, W >= 1, else ValueError (image.py:48-55)."""
    shape = _dev.shape_of(img)
    if shape is None or len(shape) != 2 or not (isinstance(img, np.ndarray) or _dev.is_tensor(img)):
        raise ValueError(f"grayscale image must have shape (H, W); got {shape}")
    if not _dev.is_u8(img):
        raise ValueError(f"luminance samples must be uint8; got {_dev.dtype_name(img)}")
    if shape[0] < 1 or shape[1] < 1:
        raise ValueError("image must be at least 1x1")
    return img


def to_grayscale(img):
    """(54 R + 183 G + 19 B) >> 8 per pixel, on the device (image.py:58-68)."""
    validate_rgb(img)
    torch = _dev.torch_mod()
    src = _dev.to_device(img)
    h, w = int(src.shape[0]), int(src.shape[1])
    out = torch.empty((h, w), dtype=torch.uint8, device=src.device)
    _lib.call("mtb_to_grayscale", _dev.ptr(src), 3 * w, 3 * w * h, w, h, 1,
              _dev.ptr(out), w, w * h, _dev.stream())
    return _dev.like_input(out, img)


def _clamp_offset(dx: int, dy: int, w: int, h: int):
    """Any integer offset, clamped to [-(w+1), w+1] x [-(h+1), h+1]: beyond the
    raster every pixel is fill either way (image.py:82-106 accepts any int), and
    the clamp keeps the values inside the kernels' int32 arithmetic."""
    return max(-(w + 1), min(w + 1, int(dx))), max(-(h + 1), min(h + 1, int(dy)))


def _offsets_tensor(offsets, w: int, h: int):
    torch = _dev.torch_mod()
    arr = np.asarray([_clamp_offset(o[0], o[1], w, h) for o in offsets], dtype=np.int32).reshape(-1, 2)
    return torch.from_numpy(arr).to("cuda")


def shift_rgb_device(batch, offsets, fill=(0, 0, 0), out=None):
    """Batched shift of an (N, H, W, 3) CUDA tensor by per-image offsets.

    offsets: (N, 2) int32 CUDA tensor or a sequence of (dx, dy).
    """
    torch = _dev.torch_mod()
    n, h, w = int(batch.shape[0]), int(batch.shape[1]), int(batch.shape[2])
    if not _dev.is_tensor(offsets):
        offsets = _offsets_tensor(offsets, w, h)
    offsets = offsets.to(torch.int32).contiguous()
    if out is None:
        out = torch.empty_like(batch)
    fr, fg, fb = (int(v) for v in fill)
    _lib.call("mtb_shift_rgb", _dev.ptr(batch), 3 * w, 3 * w * h, w, h, n, _dev.ptr(offsets),
              fr, fg, fb, _dev.ptr(out), 3 * w, 3 * w * h, _dev.stream())
    return out


def shift_rgb(img, offset: ShiftOffset, fill=(0, 0, 0)):
    """Translate an RGB raster, filling vacated pixels (image.py:82-93)."""
    validate_rgb(img)
    src = _dev.to_device(img)
    fill = tuple(int(v) for v in np.broadcast_to(np.asarray(fill, dtype=np.int64), (3,)))
    out = shift_rgb_device(src.unsqueeze(0), [offset], fill)[0]
    return _dev.like_input(out, img)


def shift_gray(img, offset: ShiftOffset, fill: int = 0):
    """Translate a grayscale raster (image.py:96-106)."""
    validate_gray(img)
    torch = _dev.torch_mod()
    src = _dev.to_device(img)
    h, w = int(src.shape[0]), int(src.shape[1])
    out = torch.empty_like(src)
    dx, dy = _clamp_offset(offset[0], offset[1], w, h)
    _lib.call("mtb_shift_gray", _dev.ptr(src), w, w, h, dx, dy, int(fill) & 0xFF, _dev.ptr(out), w, _dev.stream())
    return _dev.like_input(out, img)
