"""Shift search on the GPU: 9-candidate level search, coarse-to-fine descent
and the exhaustive oracle (mirror of mtbalign.search, search.py:1-119).

The offset returned is the correction for the TARGET: translating the target
by it minimises masked MTB disagreement with the reference.  One level adds
one bit of range, so L levels reach +-(2^L - 1) in 9L error tests.  All error
counts and the (err, |ddx|+|ddy|, index) tie-break run on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .bitmap import check_quad
from .image import ShiftOffset
from .instrumentation import FIND_OFFSET_CALLS, SHIFTED_ERROR_EVALS, counters

# search.py:20-23 — row-major (ddy, ddx) scan; the position is the last tie-break key.
NEIGHBORHOOD = tuple((ddy, ddx) for ddy in (-1, 0, 1) for ddx in (-1, 0, 1))


@dataclass(frozen=True)
class LevelTrace:
    """One level's search record, offsets at that level's scale (search.py:26-33)."""

    level: int
    candidates: list
    chosen: ShiftOffset
    accumulated: ShiftOffset


@dataclass(frozen=True)
class AlignmentResult:
    """Level-0 offset and per-level traces, deepest first (search.py:36-42)."""

    offset: ShiftOffset
    traces: list
    total_tests: int


def _check_pair_shapes(ref, tgt) -> None:
    if not ref.mtb.same_shape(tgt.mtb):
        raise ValueError(f"reference is {ref.mtb.width}x{ref.mtb.height} but target is "
                         f"{tgt.mtb.width}x{tgt.mtb.height}")


def _level_table(ref_pairs, tgt_pairs):
    """Device pointer table [n][1][4] and host dims [n][3] for one pair of pyramids."""
    torch = _dev.torch_mod()
    n = len(ref_pairs)
    table = np.empty((n, 1, 4), dtype=np.int64)
    dims = np.empty((n, 3), dtype=np.int32)
    keep = []
    for k, (r, t) in enumerate(zip(ref_pairs, tgt_pairs)):
        maps = [r.mtb.words, r.exclusion.words, t.mtb.words, t.exclusion.words]
        maps = [m if m.is_contiguous() else m.contiguous() for m in maps]
        keep.extend(maps)
        table[k, 0] = [m.data_ptr() for m in maps]
        dims[k] = (r.mtb.width, r.mtb.height, maps[0].shape[1])
    return torch.from_numpy(table).to("cuda"), np.ascontiguousarray(dims), keep


def _run_levels(ref_pairs, tgt_pairs, base):
    torch = _dev.torch_mod()
    n = len(ref_pairs)
    table, dims, keep = _level_table(ref_pairs, tgt_pairs)
    acc = torch.empty((1, n, 2), dtype=torch.int32, device="cuda")
    errs = torch.empty((1, n, 9), dtype=torch.int64, device="cuda")
    done = torch.empty((1, n), dtype=torch.int32, device="cuda")
    base_dev = None
    if base is not None:
        base_dev = torch.tensor([[int(base[0]), int(base[1])]], dtype=torch.int32, device="cuda")
    _lib.call("mtb_find_offset_batch", _dev.ptr(table), dims.ctypes.data, n, 1,
              _dev.ptr(base_dev) if base_dev is not None else None, _dev.ptr(acc), _dev.ptr(errs), _dev.ptr(done),
              _dev.stream())
    acc_h, errs_h = acc.cpu().numpy()[0], errs.cpu().numpy()[0]
    del keep
    return acc_h, errs_h


def search_level(ref, tgt, base: ShiftOffset):
    """Test base + {-1,0,1}^2 and keep the lowest error (search.py:53-71).

    Ties prefer the smaller |ddx|+|ddy|, then the earlier scan position.
    """
    _check_pair_shapes(ref, tgt)
    check_quad(ref.mtb, ref.exclusion, tgt.mtb, tgt.exclusion)
    counters.bump(SHIFTED_ERROR_EVALS, len(NEIGHBORHOOD))
    acc, errs = _run_levels([ref], [tgt], base)
    candidates = [(ShiftOffset(base.dx + ddx, base.dy + ddy), int(errs[0, i]))
                  for i, (ddy, ddx) in enumerate(NEIGHBORHOOD)]
    return ShiftOffset(int(acc[0, 0]), int(acc[0, 1])), candidates


def find_offset(ref_pairs: list, tgt_pairs: list) -> AlignmentResult:
    """Coarse-to-fine descent over two MTB pyramids, index 0 = full resolution
    (search.py:74-95); every level runs on the device back to back."""
    if len(ref_pairs) != len(tgt_pairs):
        raise ValueError("both pyramids must have the same number of levels")
    if not ref_pairs:
        raise ValueError("a pyramid needs at least one level")
    for r, t in zip(ref_pairs, tgt_pairs):
        _check_pair_shapes(r, t)
        check_quad(r.mtb, r.exclusion, t.mtb, t.exclusion)
    counters.bump(FIND_OFFSET_CALLS)
    n = len(ref_pairs)
    counters.bump(SHIFTED_ERROR_EVALS, len(NEIGHBORHOOD) * n)
    acc, errs = _run_levels(ref_pairs, tgt_pairs, None)
    traces = []
    accumulated = ShiftOffset(0, 0)
    for level in reversed(range(n)):
        base = accumulated.scaled(2)
        candidates = [(ShiftOffset(base.dx + ddx, base.dy + ddy), int(errs[level, i]))
                      for i, (ddy, ddx) in enumerate(NEIGHBORHOOD)]
        accumulated = ShiftOffset(int(acc[level, 0]), int(acc[level, 1]))
        traces.append(LevelTrace(level=level, candidates=candidates, chosen=accumulated, accumulated=accumulated))
    return AlignmentResult(offset=accumulated, traces=traces, total_tests=len(NEIGHBORHOOD) * n)


def brute_force_offset(ref, tgt, max_radius: int):
    """Exhaustive (2r+1)^2 search with the level search's tie-break measured
    from (0, 0) (search.py:98-119): all candidates in one device launch."""
    _check_pair_shapes(ref, tgt)
    check_quad(ref.mtb, ref.exclusion, tgt.mtb, tgt.exclusion)
    if max_radius < 0:
        raise ValueError("max_radius must be >= 0")
    torch = _dev.torch_mod()
    r = int(max_radius)
    offs = np.array([(dx, dy) for dy in range(-r, r + 1) for dx in range(-r, r + 1)], dtype=np.int32)
    k = len(offs)
    counters.bump(SHIFTED_ERROR_EVALS, k)
    offs_dev = torch.from_numpy(offs).to("cuda")
    errs = torch.empty(k, dtype=torch.int64, device="cuda")
    chosen = torch.empty(3, dtype=torch.int32, device="cuda")
    maps = [m.words.contiguous() for m in (ref.mtb, ref.exclusion, tgt.mtb, tgt.exclusion)]
    h, nw = int(maps[0].shape[0]), int(maps[0].shape[1])
    _lib.call("mtb_shifted_error_multi", *(_dev.ptr(m) for m in maps), h, nw, _dev.ptr(offs_dev), k,
              _dev.ptr(errs), _dev.stream())
    _lib.call("mtb_select_candidate", _dev.ptr(errs), _dev.ptr(offs_dev), k, 0, 0, _dev.ptr(chosen), _dev.stream())
    c = chosen.cpu().numpy()
    return ShiftOffset(int(c[0]), int(c[1])), int(errs[int(c[2])].item())
