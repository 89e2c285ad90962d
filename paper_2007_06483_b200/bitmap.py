"""Device-resident binary rasters and the fused shifted-error test.

Mirrors mtbalign.bitmap (pkg/src/mtbalign/bitmap.py).  Every Bitmap is
stored on the GPU in the reference's packed layout (bitmap.py:32-40): per row
ceil(W/64) u64 words, pixel x at bit x&63 of word x>>6, zero padding bits.
The `layout` attribute keeps the reference's two logical layouts; they give
identical results by contract (bitmap.py:1-8), so BYTEMAP is a view format:
`Bitmap.buf` returns the 0/255 byte map for it and the u64 word array for
PACKED, each bit-identical to what the reference would hold.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _lib, kernels
from .image import ShiftOffset
from .instrumentation import SHIFTED_ERROR_EVALS, counters

BYTEMAP = "bytemap"
PACKED = "packed"
LAYOUTS = (BYTEMAP, PACKED)

_WORD_BITS = 64


def _check_layout(layout: str) -> str:
    if layout not in LAYOUTS:
        raise ValueError(f"bitmap layout must be one of {LAYOUTS}, got {layout!r}")
    return layout


def words_per_row(width: int) -> int:
    return (int(width) + _WORD_BITS - 1) // _WORD_BITS


def pack_device(mask_dev, width: int, height: int):
    """Pack a (H, W) uint8 CUDA tensor (nonzero = set) into (H, nw64) int64 words."""
    torch = _dev.torch_mod()
    words = torch.empty((height, words_per_row(width)), dtype=torch.int64, device="cuda")
    _lib.call("mtb_pack_mask", _dev.ptr(mask_dev), int(mask_dev.stride(0)), width, height,
              _dev.ptr(words), _dev.stream())
    return words


def unpack_device(words, width: int, height: int, on_value: int):
    torch = _dev.torch_mod()
    cells = torch.empty((height, width), dtype=torch.uint8, device="cuda")
    _lib.call("mtb_unpack_bits", _dev.ptr(words), int(words.shape[1]), width, height,
              _dev.ptr(cells), width, int(on_value), _dev.stream())
    return cells


class Bitmap:
    """Immutable binary raster held on the device (construct via from_bool).

    `words` is the device (H, ceil(W/64)) int64 tensor of packed words (a view
    into an arena when produced by the fused engine).
    """

    __slots__ = ("width", "height", "layout", "words", "_host")

    def __init__(self, width: int, height: int, layout: str, buf):
        _check_layout(layout)
        self.width = int(width)
        self.height = int(height)
        self.layout = layout
        self._host = None
        if isinstance(buf, np.ndarray):
            buf = np.asarray(buf)
            if buf.dtype == np.uint64 and buf.shape == (self.height, words_per_row(self.width)):
                torch = _dev.torch_mod()
                self.words = torch.from_numpy(np.ascontiguousarray(buf).view(np.int64)).to("cuda")
            elif buf.shape == (self.height, self.width):
                self.words = pack_device(_dev.to_device((buf != 0).astype(np.uint8)), self.width, self.height)
            else:
                raise ValueError(f"buffer of shape {buf.shape} does not describe a {width}x{height} bitmap")
        else:
            self.words = buf  # device int64 (H, nw64) words

    @classmethod
    def from_bool(cls, mask, layout: str = PACKED) -> "Bitmap":
        """Bitmap of per-pixel truth values; any nonzero is true (bitmap.py:59-72)."""
        _check_layout(layout)
        if _dev.ndim_of(mask) != 2:
            raise ValueError(f"mask must be 2-D (H, W); got shape {_dev.shape_of(mask)}")
        torch = _dev.torch_mod()
        if isinstance(mask, np.ndarray):
            m = _dev.to_device(mask.astype(bool).view(np.uint8) if mask.dtype == bool
                               else (mask != 0).view(np.uint8))
        else:
            m = _dev.to_device(mask)
            if m.dtype != torch.uint8:
                m = (m != 0).to(torch.uint8)
        h, w = int(m.shape[0]), int(m.shape[1])
        if h < 1 or w < 1:
            raise ValueError("mask must be at least 1x1")
        return cls(w, h, layout, pack_device(m, w, h))

    # -- host views ---------------------------------------------------------
    @property
    def buf(self) -> np.ndarray:
        """Read-only host copy in the reference's physical layout."""
        if self._host is None:
            if self.layout == BYTEMAP:
                host = unpack_device(self.words, self.width, self.height, 255).cpu().numpy()
            else:
                host = self.words.cpu().numpy().view(np.uint64)
            host.setflags(write=False)
            self._host = host
        return self._host

    def get(self, x: int, y: int) -> bool:
        if not (0 <= x < self.width and 0 <= y < self.height):
            raise IndexError(f"({x}, {y}) is outside the {self.width}x{self.height} bitmap")
        if self.layout == BYTEMAP:
            return bool(self.buf[y, x])
        return bool((int(self.buf[y, x >> 6]) >> (x & 63)) & 1)

    def count_ones(self) -> int:
        """Set pixels (padding bits are zero and never counted), on the device."""
        return kernels.active().count_ones_packed(self.words)

    def to_bool(self) -> np.ndarray:
        return unpack_device(self.words, self.width, self.height, 1).cpu().numpy().astype(bool)

    def same_shape(self, other: "Bitmap") -> bool:
        return self.width == other.width and self.height == other.height

    def __repr__(self):
        return f"Bitmap({self.width}x{self.height}, {self.layout}, device)"


def check_quad(mtb_a: Bitmap, eb_a: Bitmap, mtb_b: Bitmap, eb_b: Bitmap) -> None:
    for m in (eb_a, mtb_b, eb_b):
        if not mtb_a.same_shape(m):
            raise ValueError("the four bitmaps must have identical dimensions")
        if m.layout != mtb_a.layout:
            raise ValueError("the four bitmaps must use one layout")


def shifted_error(mtb_a: Bitmap, eb_a: Bitmap, mtb_b: Bitmap, eb_b: Bitmap, offset: ShiftOffset) -> int:
    """Masked MTB disagreement of b translated by offset against a (bitmap.py:102-123).

    Out-of-bounds reads of the translated map contribute nothing.  One fused
    XOR/AND/popcount pass on the device.
    """
    check_quad(mtb_a, eb_a, mtb_b, eb_b)
    counters.bump(SHIFTED_ERROR_EVALS)
    return kernels.active().shifted_error_packed(mtb_a.words, eb_a.words, mtb_b.words, eb_b.words,
                                                 int(offset[0]), int(offset[1]))
