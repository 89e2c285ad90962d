"""The CUDA engine: the four-function engine contract of the reference.

Replaces kernels/_native.pyx:32,41,73,114 (and the numpy twins in
kernels/fallback.py).  Buffers may be numpy arrays laid out exactly as the
reference's (packed: (H, nwords) uint64; bytemap: (H, W) uint8) or CUDA
tensors with the same shape (int64 words for packed).  Results are Python
ints, as the reference returns.
"""

from __future__ import annotations

import numpy as np

from .. import _dev, _lib


def library_path() -> str:
    return _lib.LIB_PATH


def _words(buf):
    if isinstance(buf, np.ndarray):
        buf = np.ascontiguousarray(buf)
        if buf.dtype != np.uint64 or buf.ndim != 2:
            raise ValueError(f"packed buffers are 2-D uint64 arrays; got {buf.dtype} {buf.shape}")
        buf = buf.view(np.int64)
    return _dev.to_device(buf)


def _cells(buf):
    if isinstance(buf, np.ndarray):
        buf = np.ascontiguousarray(buf)
        if buf.dtype != np.uint8 or buf.ndim != 2:
            raise ValueError(f"byte-map buffers are 2-D uint8 arrays; got {buf.dtype} {buf.shape}")
    return _dev.to_device(buf)


def _scalar():
    torch = _dev.torch_mod()
    return torch.zeros(1, dtype=torch.int64, device="cuda")


def count_ones_packed(words) -> int:
    w = _words(words)
    out = _scalar()
    _lib.call("mtb_count_ones_packed", _dev.ptr(w), int(w.shape[0]), int(w.shape[1]), _dev.ptr(out), _dev.stream())
    return int(out.item())


def count_ones_bytemap(cells) -> int:
    c = _cells(cells)
    out = _scalar()
    _lib.call("mtb_count_ones_bytemap", _dev.ptr(c), int(c.shape[0]), int(c.shape[1]), int(c.shape[1]),
              _dev.ptr(out), _dev.stream())
    return int(out.item())


def shifted_error_packed(a, ea, b, eb, dx: int, dy: int) -> int:
    maps = [_words(m) for m in (a, ea, b, eb)]
    h, nw = int(maps[0].shape[0]), int(maps[0].shape[1])
    for m in maps[1:]:
        if tuple(m.shape) != (h, nw):
            raise ValueError("packed buffers must share one shape")
    out = _scalar()
    _lib.call("mtb_shifted_error_packed", *(_dev.ptr(m) for m in maps), h, nw, int(dx), int(dy),
              _dev.ptr(out), _dev.stream())
    return int(out.item())


def shifted_error_bytemap(a, ea, b, eb, dx: int, dy: int) -> int:
    maps = [_cells(m) for m in (a, ea, b, eb)]
    h, w = int(maps[0].shape[0]), int(maps[0].shape[1])
    for m in maps[1:]:
        if tuple(m.shape) != (h, w):
            raise ValueError("byte-map buffers must share one shape")
    out = _scalar()
    _lib.call("mtb_shifted_error_bytemap", *(_dev.ptr(m) for m in maps), h, w, w, int(dx), int(dy),
              _dev.ptr(out), _dev.stream())
    return int(out.item())
