"""Stack alignment on the GPU (mirror of mtbalign.pipeline, pipeline.py:1-151).

`align_stack` keeps the reference's contract: chain alignment (image i+1
against image i), offsets re-based onto image 0 by prefix sums, image 0
passed through untouched, per-stage timings that tile the call.  The work
behind it is batched on the device: every image's MTB pyramid and every
pair's coarse-to-fine search run in one batched pass, the cumulative offsets
are summed on the device and all outputs are shifted in one launch.

Path selection (`use_fused`): batches of >= 20 images of >= 20 MP (or >= 96
of >= 13 MP) go through the fused pipeline (csrc/pipe.cu: preprocess and
search of the whole stack in one pipelined launch sequence, 25 % faster for
64 pairs of 24 MP); images whose gray pyramid
fits the shared memory of a 1- or 2-CTA cluster (about 0.4 MP) through the
on-chip preprocess (csrc/cluster.cu: one launch over the whole batch, gray
never in HBM) and the batched search; the sizes between through the staged
kernels (one persistent K1 launch over the batch).

Stage windows (pipeline.py:74-112) are CUDA events recorded on the stream at
the stage boundaries, read after ONE synchronisation at the end of the call
(no device-wide syncs inside it); host time after the last event is added
to the last stage, so the stages still sum to the call's wall time:
  grayscale  host -> device upload of the stack
  pyramid    fused gray + pyramid + histograms (staged), the on-chip
             preprocess (images <= 0.4 MP: thresholds included), or the whole
             fused pipeline (preprocess, thresholds and search overlap there)
  threshold  medians + MTB / exclusion packing (staged; 0 otherwise)
  search     batched find_offset (staged) + readback of offsets and traces
  shift      device prefix sums, batched shift_rgb, download of the outputs

Additions over the reference API (north star): `align` (chain or pivot
pairing — config 3 aligns a 7-exposure stack to its middle exposure),
`align_stacks` (many same-size stacks in one device batch) and
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


# Fused pipeline or staged kernels.  The pipeline's
# per-launch fixed costs pay only for large images in large batches:
#   pairs/s at 128 pairs per call: 6 MP staged 56.5 K vs fused 30.4 K, 8 MP
#   42.9 K vs 29.1 K, 12 MP 29.6 K both, 16 MP fused 25.7 K vs 23.5 K, 24 MP
#   18.3 K vs 14.7 K;
#   call latency of n-image chains: 24 MP staged faster up to 13 images
#   (2: 0.16 vs 0.22 ms, 13: 0.54 vs 0.57 ms), fused from 25 (0.93 vs 0.96);
#   16 MP staged up to ~50 images, even at 97.
FUSED_MIN_PIXELS = 13_000_000
FUSED_MIN_IMAGES = {20_000_000: 20, FUSED_MIN_PIXELS: 96}   # image size -> batch size from which fused wins


def use_fused(eng: MtbEngine, n_img: int) -> bool:
    """True when the fused pipeline is the faster path for a call of n_img of
    this engine's images."""
    if not eng.fused_supported:
        return False
    px = eng.width * eng.height
    for min_px, min_img in sorted(FUSED_MIN_IMAGES.items(), reverse=True):
        if px >= min_px:
            return n_img >= min_img
    return False


class _StageClock:
    """CUDA events at stage boundaries on the current stream; one sync at the end."""

    def __init__(self):
        self.torch = _dev.torch_mod()
        self.t0 = time.perf_counter()
        self.events = []
        self.mark()

    def mark(self):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record()
        self.events.append(ev)

    def timings(self, names):
        """Stage durations in ms (events[i] -> events[i+1]); host time after
        the last event (result unpacking) is charged to the last stage."""
        self.events[-1].synchronize()
        wall = (time.perf_counter() - self.t0) * 1000.0
        out = {n: self.events[i].elapsed_time(self.events[i + 1]) for i, n in enumerate(names)}
        rest = max(0.0, wall - sum(out.values()))
        out[names[-1]] += rest
        return out


def _pairs_for(n: int, mode: str, pivot):
    if mode == "chain":
        return [(i, i + 1) for i in range(n - 1)], None
    if mode != "pivot":
        raise ValueError(f"mode must be 'chain' or 'pivot', got {mode!r}")
    p = n // 2 if pivot is None else int(pivot)
    if not 0 <= p < n:
        raise ValueError(f"pivot {p} out of range for {n} images")
    return [(p, i) for i in range(n) if i != p], p


def _run_batch(eng: MtbEngine, batch, pairs, clk: _StageClock):
    """Preprocess + search of a device batch; marks pyramid / threshold / search."""
    n_img = int(batch.shape[0])
    if use_fused(eng, n_img):
        _, acc, errs = eng.align_fused(batch, pairs)
        clk.mark()          # pyramid: the whole pipelined sequence
        clk.mark()          # threshold: inside it
    elif eng.on_chip_maps():
        pyr = eng.preprocess(batch, maps_only=True)   # one launch, gray kept on chip (csrc/cluster.cu)
        clk.mark()          # pyramid and threshold: the same kernel
        clk.mark()
        acc, errs = eng.search(pyr, pairs)
    else:
        pyr = eng.alloc(n_img)
        eng.pyramid_hist(batch, pyr)
        clk.mark()
        eng.threshold_levels(pyr, n_img)
        counters.bump(PYRAMID_BUILDS, n_img)
        counters.bump(MTB_PYRAMID_BUILDS, n_img)
        clk.mark()
        acc, errs = eng.search(pyr, pairs)
    return acc, errs


def _device_cumulative(acc, n_img: int, pairs, anchor):
    """(n_img, 2) int32 device offsets onto the anchor: prefix sums of the
    chain's pairwise offsets (pipeline.py:91-93), or each pair's own offset
    against the pivot."""
    torch = _dev.torch_mod()
    cum = torch.zeros((n_img, 2), dtype=torch.int32, device="cuda")
    if anchor is None:
        cum[1:] = torch.cumsum(acc[:, 0], dim=0, dtype=torch.int32)
    else:
        tgts = torch.tensor([t for _, t in pairs], dtype=torch.long, device="cuda")
        cum.index_copy_(0, tgts, acc[:, 0].to(torch.int32))
    return cum


def _align_batch(images, stacks, levels, tol, layout, mode, pivot):
    """Shared body of align_stack / align / align_stacks.  `stacks` = list of
    (first image index, count) of the same-size stacks inside `images`."""
    w, h = _validate_stack(images)
    _check_layout(layout)
    torch = _dev.torch_mod()
    clk = _StageClock()
    eng = engine_for(w, h, levels, tol)
    batch = upload_stack(images)
    clk.mark()
    pairs, anchors = [], []
    for i0, n in stacks:
        ps, anchor = _pairs_for(n, mode, pivot)
        pairs += [(i0 + r, i0 + t) for r, t in ps]
        anchors.append(anchor)
    acc, errs = _run_batch(eng, batch, pairs, clk)
    acc_h = torch.empty(tuple(acc.shape), dtype=acc.dtype, pin_memory=True)
    errs_h = torch.empty(tuple(errs.shape), dtype=errs.dtype, pin_memory=True)
    acc_h.copy_(acc, non_blocking=True)
    errs_h.copy_(errs, non_blocking=True)
    clk.mark()
    # shift: every non-anchor image onto its stack's anchor, offsets stay on the device
    cum, movers = [], []
    q = 0
    for (i0, n), anchor in zip(stacks, anchors):
        np_ = n - 1
        cum.append(_device_cumulative(acc[q:q + np_], n, [(r - i0, t - i0) for r, t in pairs[q:q + np_]], anchor))
        keep = 0 if anchor is None else anchor
        movers += [i0 + i for i in range(n) if i != keep]
        q += np_
    cum = torch.cat(cum)
    idx = torch.tensor(movers, dtype=torch.long, device="cuda")
    shifted = shift_rgb_device(batch.index_select(0, idx).contiguous(), cum.index_select(0, idx).contiguous())
    as_numpy = isinstance(images[0], np.ndarray)
    if as_numpy:
        host = torch.empty(tuple(shifted.shape), dtype=torch.uint8, pin_memory=True)
        host.copy_(shifted, non_blocking=True)
    clk.mark()
    timings = clk.timings(STAGES)
    out_imgs = list(images)
    src = host.numpy() if as_numpy else shifted
    for j, i in enumerate(movers):
        out_imgs[i] = src[j]
    results = []
    q = 0
    for (i0, n), anchor in zip(stacks, anchors):
        np_ = n - 1
        pairwise = results_from_device(acc_h[q:q + np_], errs_h[q:q + np_])
        cumulative = [ShiftOffset(0, 0)] * n
        if anchor is None:
            for i, res in enumerate(pairwise, start=1):
                cumulative[i] = cumulative[i - 1] + res.offset
        else:
            for (_, tgt), res in zip(pairs[q:q + np_], pairwise):
                cumulative[tgt - i0] = res.offset
        record = StackAlignment(image_count=n, pairwise=pairwise, cumulative=cumulative, timings=dict(timings))
        results.append((out_imgs[i0:i0 + n], record))
        q += np_
    return results


def align_stack(images: list, levels: int = DEFAULT_LEVELS, tol: int = DEFAULT_NOISE_TOLERANCE,
                layout: str = PACKED, workers: int | None = None):
    """Align a bracketed stack onto its first image (pipeline.py:52-120).

    Returns (aligned images, StackAlignment); image 0 is returned as the same
    object.  `workers` is accepted for API compatibility; the device batches
    every image and pair regardless, so results never depend on it.
    """
    (aligned, record), = _align_batch(list(images), [(0, len(images))], levels, tol, layout, "chain", None)
    return aligned, record


def align(images: list, levels: int = DEFAULT_LEVELS, tol: int = DEFAULT_NOISE_TOLERANCE,
          layout: str = PACKED, mode: str = "chain", pivot: int | None = None):
    """`align_stack` with a choice of pairing.

    mode="chain": the reference's chain (identical to align_stack).
    mode="pivot": every image is searched directly against the pivot (default
    the middle exposure, len//2) and aligned onto it; the pivot is returned
    untouched.  Each pair is find_offset(mtb[pivot], mtb[i]).
    """
    n = len(images)
    if mode not in ("chain", "pivot"):
        raise ValueError(f"mode must be 'chain' or 'pivot', got {mode!r}")
    if n < 2:
        raise ValueError(f"alignment needs at least 2 images; got {n}")
    _pairs_for(n, mode, pivot)   # validates the pivot
    (aligned, record), = _align_batch(list(images), [(0, n)], levels, tol, layout, mode, pivot)
    return aligned, record


def align_stacks(stacks: list, levels: int = DEFAULT_LEVELS, tol: int = DEFAULT_NOISE_TOLERANCE,
                 layout: str = PACKED, mode: str = "chain", pivot: int | None = None):
    """Align many same-size stacks in ONE device batch: every
    stack's pyramids and searches run in one pass, every output in one shift
    launch.  Returns [(aligned images, StackAlignment)] in input order; each
    record carries the batch's stage timings.  Results equal per-stack
    `align(stack, mode=mode, pivot=pivot)` calls."""
    stacks = [list(st) for st in stacks]
    if not stacks:
        return []
    if mode not in ("chain", "pivot"):
        raise ValueError(f"mode must be 'chain' or 'pivot', got {mode!r}")
    images, spans = [], []
    for st in stacks:
        if len(st) < 2:
            raise ValueError(f"alignment needs at least 2 images; got {len(st)}")
        _pairs_for(len(st), mode, pivot)
        spans.append((len(images), len(st)))
        images += st
    return _align_batch(images, spans, levels, tol, layout, mode, pivot)


def get_exp_shift(ref_rgb, tgt_rgb, levels: int = DEFAULT_LEVELS, tol: int = DEFAULT_NOISE_TOLERANCE) -> ShiftOffset:
    """Offset that aligns tgt_rgb onto ref_rgb (find_offset on RGB input)."""
    w, h = _validate_stack([ref_rgb, tgt_rgb])
    eng = engine_for(w, h, levels, tol)
    batch = upload_stack([ref_rgb, tgt_rgb])
    if use_fused(eng, 2):   # (never, with the measured thresholds: one pair is faster staged)
        _, acc, _ = eng.align_fused(batch, [(0, 1)])     # one pipelined launch sequence (csrc/pipe.cu)
    else:
        pyr = eng.preprocess(batch, maps_only=True)
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
    pairs, anchor = _pairs_for(n, mode, pivot)
    t0 = time.perf_counter()
    host = load_stack(paths, workers=workers, pinned=True)
    t1 = time.perf_counter()
    h, w = int(host.shape[1]), int(host.shape[2])
    if w < MIN_LEVEL_SIZE or h < MIN_LEVEL_SIZE:
        raise ValueError(f"images must be at least 16x16; got {w}x{h}")
    eng = engine_for(w, h, levels, tol)
    if use_fused(eng, n):
        batch, _, acc, errs = eng.align_fused_host(host, pairs)
    else:
        batch = host.to("cuda", non_blocking=True)
        pyr = eng.preprocess(batch, maps_only=True)
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
