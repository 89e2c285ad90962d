"""Stack alignment on the GPU (mirror of mtbalign.pipeline, pipeline.py:1-151).

`align_stack` keeps the reference's contract: chain alignment (image i+1
against image i), offsets re-based onto image 0 by prefix sums, image 0
passed through untouched, per-stage timings that tile the call.  The work
behind it is batched on the device: every image's MTB pyramid is built by
one fused preprocess over the whole stack, all N-1 searches run as one
batched coarse-to-fine search, and all outputs are shifted in one launch.

Stage windows (host wall clock, synchronised at each boundary):
  grayscale  host -> device upload of the stack
  pyramid    fused gray + pyramid + per-level histograms (one RGB pass)
  threshold  medians + MTB / exclusion packing of every level
  search     batched find_offset + readback of offsets and traces
  shift      batched shift_rgb + download of the aligned images

Additions over the reference API (north star): `align` (chain or pivot
pairing — config 3 aligns a 7-exposure stack to its middle exposure) and
`get_exp_shift` (one pair; OpenCV/Ward naming of find_offset on RGB input).
"""

from __future__ import annotations

import statistics
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import _dev
from .bitmap import PACKED, _check_layout
from .engine import MtbEngine, results_from_device
from .image import ShiftOffset, shift_rgb_device, validate_rgb
from .instrumentation import MTB_PYRAMID_BUILDS, PYRAMID_BUILDS, counters
from .pyramid import DEFAULT_LEVELS, MIN_LEVEL_SIZE
from .search import AlignmentResult
from .threshold import DEFAULT_NOISE_TOLERANCE

STAGES = ("grayscale", "pyramid", "threshold", "search", "shift")


@dataclass(frozen=True)
class StackAlignment:
    """Offsets and timings for one aligned stack (pipeline.py:29-36)."""

    image_count: int
    pairwise: list
    cumulative: list
    timings: dict


@dataclass(frozen=True)
class StageStats:
    mean_ms: float
    stddev_ms: float


@dataclass(frozen=True)
class TimingReport:
    repetitions: int
    stages: dict
    total: StageStats


_engines: dict = {}
_engines_mu = threading.Lock()


def engine_for(width: int, height: int, levels: int, tol: int) -> MtbEngine:
    key = (int(width), int(height), int(levels), int(tol))
    with _engines_mu:
        eng = _engines.get(key)
        if eng is None:
            eng = MtbEngine(width, height, levels, tol)
            if len(_engines) > 16:
                _engines.clear()
            _engines[key] = eng
        return eng


def _validate_stack(images):
    if len(images) < 2:
        raise ValueError(f"alignment needs at least 2 images; got {len(images)}")
    for img in images:
        validate_rgb(img)
    h, w = _dev.shape_of(images[0])[:2]
    for i, img in enumerate(images[1:], start=1):
        if _dev.shape_of(img)[:2] != (h, w):
            s = _dev.shape_of(img)
            raise ValueError(f"image {i} is {s[1]}x{s[0]} but image 0 is {w}x{h}")
    if w < MIN_LEVEL_SIZE or h < MIN_LEVEL_SIZE:
        raise ValueError(f"images must be at least 16x16; got {w}x{h}")
    return w, h


def upload_stack(images):
    """(N, H, W, 3) contiguous CUDA batch of the images (pinned staging for numpy)."""
    torch = _dev.torch_mod()
    if all(_dev.is_tensor(im) and im.is_cuda for im in images):
        return torch.stack([im.contiguous() for im in images])
    h, w = _dev.shape_of(images[0])[:2]
    host = torch.empty((len(images), h, w, 3), dtype=torch.uint8, pin_memory=True)
    hv = host.numpy()
    for i, im in enumerate(images):
        if isinstance(im, np.ndarray):
            hv[i] = im
        else:
            host[i].copy_(im)
    return host.to("cuda", non_blocking=True)


def _sync():
    _dev.torch_mod().cuda.synchronize()


def _align(images, pairs, levels, tol, layout, pivot):
    """Shared body of align_stack / align: pairs are (ref, tgt) image indices."""
    w, h = _validate_stack(images)
    _check_layout(layout)
    n_img = len(images)
    timings = {}
    t0 = time.perf_counter()
    eng = engine_for(w, h, levels, tol)
    batch = upload_stack(images)
    _sync()
    t1 = time.perf_counter()
    pyr = eng.alloc(n_img)
    eng.pyramid_hist(batch, pyr)
    _sync()
    t2 = time.perf_counter()
    eng.threshold_levels(pyr, n_img)
    counters.bump(PYRAMID_BUILDS, n_img)
    counters.bump(MTB_PYRAMID_BUILDS, n_img)
    _sync()
    t3 = time.perf_counter()
    acc, errs = eng.search(pyr, pairs)
    pairwise = results_from_device(acc, errs)
    # Re-basing: chain mode sums the pairwise offsets (pipeline.py:91-93); in
    # pivot mode every pair already measures image i against the pivot.
    cumulative = [ShiftOffset(0, 0)] * n_img
    if pivot is None:
        for i, res in enumerate(pairwise, start=1):
            cumulative[i] = cumulative[i - 1] + res.offset
    else:
        for (ref, tgt), res in zip(pairs, pairwise):
            cumulative[tgt] = res.offset
    t4 = time.perf_counter()
    anchor = 0 if pivot is None else pivot
    movers = [i for i in range(n_img) if i != anchor]
    torch = _dev.torch_mod()
    idx = torch.tensor(movers, dtype=torch.long, device="cuda")
    shifted = shift_rgb_device(batch.index_select(0, idx).contiguous(), [cumulative[i] for i in movers])
    aligned = list(images)
    as_numpy = isinstance(images[0], np.ndarray)
    host = shifted.cpu().numpy() if as_numpy else shifted
    for j, i in enumerate(movers):
        aligned[i] = host[j]
    _sync()
    t5 = time.perf_counter()
    timings["grayscale"] = (t1 - t0) * 1000.0
    timings["pyramid"] = (t2 - t1) * 1000.0
    timings["threshold"] = (t3 - t2) * 1000.0
    timings["search"] = (t4 - t3) * 1000.0
    timings["shift"] = (t5 - t4) * 1000.0
    record = StackAlignment(image_count=n_img, pairwise=pairwise, cumulative=cumulative, timings=timings)
    return aligned, record


def align_stack(images: list, levels: int = DEFAULT_LEVELS, tol: int = DEFAULT_NOISE_TOLERANCE,
                layout: str = PACKED, workers: int | None = None):
    """Align a bracketed stack onto its first image (pipeline.py:52-120).

    Returns (aligned images, StackAlignment); image 0 is returned as the same
    object.  `workers` is accepted for API compatibility; the device batches
    every image and pair regardless, so results never depend on it.
    """
    n = len(images)
    return _align(images, [(i, i + 1) for i in range(n - 1)], levels, tol, layout, None)


def align(images: list, levels: int = DEFAULT_LEVELS, tol: int = DEFAULT_NOISE_TOLERANCE,
          layout: str = PACKED, mode: str = "chain", pivot: int | None = None):
    """`align_stack` with a choice of pairing.

    mode="chain": the reference's chain (identical to align_stack).
    mode="pivot": every image is searched directly against the pivot (default
    the middle exposure, len//2) and aligned onto it; the pivot is returned
    untouched.  Each pair is find_offset(mtb[pivot], mtb[i]).
    """
    n = len(images)
    if mode == "chain":
        return align_stack(images, levels, tol, layout)
    if mode != "pivot":
        raise ValueError(f"mode must be 'chain' or 'pivot', got {mode!r}")
    if n < 2:
        raise ValueError(f"alignment needs at least 2 images; got {n}")
    p = n // 2 if pivot is None else int(pivot)
    if not 0 <= p < n:
        raise ValueError(f"pivot {p} out of range for {n} images")
    return _align(images, [(p, i) for i in range(n) if i != p], levels, tol, layout, p)


def get_exp_shift(ref_rgb, tgt_rgb, levels: int = DEFAULT_LEVELS, tol: int = DEFAULT_NOISE_TOLERANCE) -> ShiftOffset:
    """Offset that aligns tgt_rgb onto ref_rgb (find_offset on RGB input)."""
    w, h = _validate_stack([ref_rgb, tgt_rgb])
    eng = engine_for(w, h, levels, tol)
    batch = upload_stack([ref_rgb, tgt_rgb])
    if eng.fused_supported:
        _, acc, _ = eng.align_fused(batch, [(0, 1)])     # one pipelined launch sequence (csrc/pipe.cu)
    else:
        pyr = eng.preprocess(batch)
        acc, _ = eng.search(pyr, [(0, 1)])
    a = acc[0, 0].cpu().numpy()
    return ShiftOffset(int(a[0]), int(a[1]))


def align_files(paths, levels: int = DEFAULT_LEVELS, tol: int = DEFAULT_NOISE_TOLERANCE, mode: str = "chain",
                pivot: int | None = None, workers: int | None = None):
    """Ingest path: decode the files (PPM / PNG, imageio.py:82-94)
    with a thread pool straight into one pinned batch, upload it image by
    image on a copy stream overlapped with the fused pipeline (K1 of image i
    starts when its copy lands), then shift every image onto the anchor.

    Same pairing and re-basing as `align` (chain: onto image 0; pivot: onto
    the pivot).  Returns (aligned numpy images, StackAlignment) with timings
    "decode" (host decode), "align" (upload + preprocess + search + readback)
    and "shift" (shift_rgb + download).
    """
    from .imageio import load_stack

    paths = list(paths)
    n = len(paths)
    if n < 2:
        raise ValueError(f"alignment needs at least 2 images; got {n}")
    if mode == "chain":
        pairs, anchor = [(i, i + 1) for i in range(n - 1)], None
    elif mode == "pivot":
        anchor = n // 2 if pivot is None else int(pivot)
        if not 0 <= anchor < n:
            raise ValueError(f"pivot {anchor} out of range for {n} images")
        pairs = [(anchor, i) for i in range(n) if i != anchor]
    else:
        raise ValueError(f"mode must be 'chain' or 'pivot', got {mode!r}")
    t0 = time.perf_counter()
    host = load_stack(paths, workers=workers, pinned=True)
    t1 = time.perf_counter()
    h, w = int(host.shape[1]), int(host.shape[2])
    if w < MIN_LEVEL_SIZE or h < MIN_LEVEL_SIZE:
        raise ValueError(f"images must be at least 16x16; got {w}x{h}")
    eng = engine_for(w, h, levels, tol)
    if eng.fused_supported:
        batch, _, acc, errs = eng.align_fused_host(host, pairs)
    else:
        batch = host.to("cuda", non_blocking=True)
        pyr = eng.preprocess(batch)
        acc, errs = eng.search(pyr, pairs)
    pairwise = results_from_device(acc, errs)
    t2 = time.perf_counter()
    cumulative = [ShiftOffset(0, 0)] * n
    if anchor is None:
        for i, res in enumerate(pairwise, start=1):
            cumulative[i] = cumulative[i - 1] + res.offset
    else:
        for (_, tgt), res in zip(pairs, pairwise):
            cumulative[tgt] = res.offset
    keep = 0 if anchor is None else anchor
    movers = [i for i in range(n) if i != keep]
    torch = _dev.torch_mod()
    idx = torch.tensor(movers, dtype=torch.long, device="cuda")
    shifted = shift_rgb_device(batch.index_select(0, idx).contiguous(), [cumulative[i] for i in movers]).cpu().numpy()
    hv = host.numpy()
    aligned = [hv[keep].copy() if i == keep else None for i in range(n)]
    for j, i in enumerate(movers):
        aligned[i] = shifted[j]
    t3 = time.perf_counter()
    timings = {"decode": (t1 - t0) * 1000.0, "align": (t2 - t1) * 1000.0, "shift": (t3 - t2) * 1000.0}
    return aligned, StackAlignment(image_count=n, pairwise=pairwise, cumulative=cumulative, timings=timings)


def measure_alignment(images: list, repetitions: int = 10, levels: int = DEFAULT_LEVELS,
                      tol: int = DEFAULT_NOISE_TOLERANCE, layout: str = PACKED,
                      workers: int | None = None) -> TimingReport:
    """Repeat align_stack on in-memory images; per-stage mean/stddev (pipeline.py:123-151)."""
    if repetitions < 1:
        raise ValueError("repetitions must be >= 1")
    samples = {name: [] for name in STAGES}
    totals = []
    for _ in range(repetitions):
        start = time.perf_counter()
        _, record = align_stack(images, levels=levels, tol=tol, layout=layout, workers=workers)
        totals.append((time.perf_counter() - start) * 1000.0)
        for name in STAGES:
            samples[name].append(record.timings[name])

    def stats(xs):
        return StageStats(mean_ms=statistics.fmean(xs), stddev_ms=statistics.stdev(xs) if len(xs) > 1 else 0.0)

    return TimingReport(repetitions=repetitions, stages={k: stats(v) for k, v in samples.items()},
                        total=stats(totals))
