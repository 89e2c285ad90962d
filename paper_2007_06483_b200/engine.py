"""Batched, device-resident MTB engine: the fused hot path.

One `MtbEngine` serves images of one size and one (levels, tol) setting.
`preprocess` runs to_grayscale -> build_pyramid -> build_mtb_pyramid for a
whole batch of RGB images in three kernels (pipeline.py:80-85 fused; see
csrc/pyramid.cu, csrc/threshold.cu).  `search` runs find_offset for any
number of (reference, target) image pairs with every level on the device
(search.py:74-95; csrc/search.cu): the offset chosen at one level feeds the
next through device memory, so nothing returns to the host until the caller
reads the results.

Arena layout in HBM (per image, from mtb_plan_levels):
  gray    level k at gray_off[k], row pitch round_up(w_k, 64) bytes
  bitmaps level k at bit_off[k] u64 words, ceil(w_k/64) words per row —
          the reference's packed layout (bitmap.py:32-40), one arena for the
          MTBs and one for the exclusion maps.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .bitmap import PACKED, Bitmap
from .image import ShiftOffset
from .instrumentation import (FIND_OFFSET_CALLS, MTB_PYRAMID_BUILDS, PYRAMID_BUILDS, SHIFTED_ERROR_EVALS,
                              counters)
from .search import NEIGHBORHOOD, AlignmentResult, LevelTrace
from .threshold import MtbPair


@dataclass
class PyramidSet:
    """Device arenas holding the MTB pyramids of a batch of images."""

    n_img: int
    gray: "object"        # uint8 [n_img, gray_image_bytes]
    hist_ws: "object"     # int32 [n_img, hist_ws_elems] (spread histograms)
    hist: "object"        # int32 [n_img, n, 256] dense histograms (or None)
    medians: "object"     # int32 [n_img, n]
    mtb: "object"         # int64 [n_img, bitmap_image_words]
    excl: "object"        # int64 [n_img, bitmap_image_words]


class MtbEngine:
    def __init__(self, width: int, height: int, levels: int = 6, tol: int = 4):
        self.torch = _dev.torch_mod()
        plan = _lib.plan_levels(width, height, levels)
        if plan is None:
            raise ValueError(f"images must be at least 16x16 and levels >= 1; got {width}x{height}, {levels}")
        self.width, self.height, self.requested_levels, self.tol = int(width), int(height), int(levels), int(tol)
        self.n, self.geom, sizes = plan
        self.gray_img_bytes = int(sizes[0])
        self.bit_img_words = int(sizes[1])
        self.hist_ws_elems = int(sizes[2])
        self.dims = np.ascontiguousarray(
            np.stack([self.geom[:, 0], self.geom[:, 1], self.geom[:, 4]], axis=1).astype(np.int32))
        self._tables = {}
        self._maps_cluster = None

    # ------------------------------------------------------------ buffers --
    def alloc(self, n_img: int, keep_hist: bool = False, gray: bool = True) -> PyramidSet:
        """Arenas for n_img images; gray=False leaves out the gray pyramid and
        histogram workspaces (enough for preprocess_maps)."""
        t = self.torch
        return PyramidSet(
            n_img=n_img,
            gray=t.empty((n_img, self.gray_img_bytes), dtype=t.uint8, device="cuda") if gray else None,
            hist_ws=t.empty((n_img, self.hist_ws_elems), dtype=t.int32, device="cuda") if gray else None,
            hist=t.empty((n_img, self.n, 256), dtype=t.int32, device="cuda") if keep_hist else None,
            medians=t.empty((n_img, self.n), dtype=t.int32, device="cuda"),
            mtb=t.empty((n_img, self.bit_img_words), dtype=t.int64, device="cuda"),
            excl=t.empty((n_img, self.bit_img_words), dtype=t.int64, device="cuda"),
        )

    def _check_rgb(self, rgb):
        t = self.torch
        if not (_dev.is_tensor(rgb) and rgb.is_cuda and rgb.dtype == t.uint8 and rgb.dim() == 4
                and tuple(rgb.shape[1:]) == (self.height, self.width, 3)):
            raise ValueError(f"expected a CUDA uint8 (N, {self.height}, {self.width}, 3) batch, got "
                             f"{getattr(rgb, 'shape', None)} {getattr(rgb, 'dtype', None)}")
        if not rgb.is_contiguous():
            raise ValueError("RGB batch must be contiguous")

    # ---------------------------------------------------------- preprocess --
    def _ptrs(self, rgb, pyr: PyramidSet, i0: int):
        """Device addresses of image i0 in the input batch and in every arena."""
        img_bytes = 3 * self.width * self.height
        return dict(
            rgb=(_dev.ptr(rgb) + i0 * img_bytes) if rgb is not None else None,
            gray=(_dev.ptr(pyr.gray) + i0 * self.gray_img_bytes) if pyr.gray is not None else None,
            hist_ws=(_dev.ptr(pyr.hist_ws) + i0 * self.hist_ws_elems * 4) if pyr.hist_ws is not None else None,
            hist=(_dev.ptr(pyr.hist) + i0 * self.n * 256 * 4) if pyr.hist is not None else None,
            medians=_dev.ptr(pyr.medians) + i0 * self.n * 4,
            mtb=_dev.ptr(pyr.mtb) + i0 * self.bit_img_words * 8,
            excl=_dev.ptr(pyr.excl) + i0 * self.bit_img_words * 8,
        )

    def pyramid_hist(self, rgb, pyr: PyramidSet, i0: int = 0, count: int | None = None):
        """Stage 1: gray + pyramid + per-level histograms (one RGB pass) of images [i0, i0+count)."""
        count = int(rgb.shape[0]) - i0 if count is None else count
        p = self._ptrs(rgb, pyr, i0)
        _lib.call("mtb_pyramid_hist", p["rgb"], 3 * self.width, 3 * self.width * self.height,
                  self.width, self.height, count, self.requested_levels, p["gray"], p["hist_ws"], _dev.stream())

    def threshold_levels(self, pyr: PyramidSet, n_img: int, i0: int = 0, discard_gray: bool = False):
        """Stage 2: medians + MTB/exclusion packing of every level of images [i0, i0+n_img).

        discard_gray drops the consumed gray lines from L2 without write-back
        (the gray arena is undefined afterwards)."""
        p = self._ptrs(None, pyr, i0)
        _lib.call("mtb_threshold_levels", p["gray"], p["hist_ws"], self.width, self.height,
                  n_img, self.requested_levels, self.tol, p["hist"], p["medians"], p["mtb"], p["excl"],
                  1 if discard_gray else 0, _dev.stream())

    def preprocess_range(self, rgb, pyr: PyramidSet, i0: int, count: int):
        """Fused preprocess (all three kernels) of images [i0, i0+count) into their arena slots."""
        p = self._ptrs(rgb, pyr, i0)
        _lib.call("mtb_preprocess", p["rgb"], 3 * self.width, 3 * self.width * self.height, self.width,
                  self.height, count, self.requested_levels, self.tol, p["gray"], p["hist_ws"], p["hist"],
                  p["medians"], p["mtb"], p["excl"], _dev.stream())

    def maps_cluster(self) -> int:
        """Cluster size of the on-chip preprocess (csrc/cluster.cu) for this
        geometry on the current device; 0 when the image does not fit one
        cluster, has more than 6 levels or its rows are not 16-byte multiples
        (TMA)."""
        if self._maps_cluster is None:
            self._maps_cluster = int(_lib.load().mtb_preprocess_maps_cluster(
                self.width, self.height, self.requested_levels)) if (3 * self.width) % 16 == 0 else 0
        return self._maps_cluster

    def on_chip_maps(self) -> bool:
        """True when preprocess(maps_only=True) takes the on-chip kernel: it
        beats the staged kernels only while an image fits a cluster of <= 2
        CTAs (about 0.4 MP; measured 1.3-1.7x there, 0.65-0.85x at 4-16 CTAs:
        DESIGN.md 4.6)."""
        return 0 < self.maps_cluster() <= 2

    def preprocess_maps(self, rgb, pyr: PyramidSet, i0: int = 0, count: int | None = None):
        """Medians + packed maps of images [i0, i0+count) without a gray arena:
        one launch, each image's gray pyramid held in a thread-block cluster's
        shared memory (requires maps_cluster() > 0)."""
        count = int(rgb.shape[0]) - i0 if count is None else count
        p = self._ptrs(rgb, pyr, i0)
        _lib.call("mtb_preprocess_maps", p["rgb"], 3 * self.width, 3 * self.width * self.height, self.width,
                  self.height, count, self.requested_levels, self.tol, p["hist"], p["medians"], p["mtb"],
                  p["excl"], _dev.stream())

    def preprocess(self, rgb, pyr: PyramidSet | None = None, keep_hist: bool = False,
                   count: bool = True, maps_only: bool = False) -> PyramidSet:
        """MTB pyramids of an (N, H, W, 3) CUDA batch (pipeline.py:80-85 fused).

        maps_only: the gray pyramid is not needed afterwards; small images then
        take the on-chip cluster kernel (no gray arena is allocated)."""
        self._check_rgb(rgb)
        n_img = int(rgb.shape[0])
        on_chip = maps_only and self.on_chip_maps()
        if pyr is None:
            pyr = self.alloc(n_img, keep_hist, gray=not on_chip)
        if on_chip:
            self.preprocess_maps(rgb, pyr, 0, n_img)
        else:
            self.preprocess_range(rgb, pyr, 0, n_img)
        if count:
            counters.bump(PYRAMID_BUILDS, n_img)
            counters.bump(MTB_PYRAMID_BUILDS, n_img)
        return pyr

    # ------------------------------------------------------------- views --
    def gray_level(self, pyr: PyramidSet, img: int, k: int):
        w, h, pitch, off = (int(v) for v in self.geom[k, :4])
        return pyr.gray[img, off:off + pitch * h].view(h, pitch)[:, :w]

    def bitmap_words(self, arena, img: int, k: int):
        w, h, nw, off = int(self.geom[k, 0]), int(self.geom[k, 1]), int(self.geom[k, 4]), int(self.geom[k, 5])
        return arena[img, off:off + nw * h].view(h, nw)

    def mtb_pyramid(self, pyr: PyramidSet, img: int, layout: str = PACKED, medians=None) -> list:
        """Reference-shaped list[MtbPair] views of one image's arena slices."""
        if medians is None:
            medians = pyr.medians[img].cpu().numpy()
        out = []
        for k in range(self.n):
            w, h = int(self.geom[k, 0]), int(self.geom[k, 1])
            out.append(MtbPair(mtb=Bitmap(w, h, layout, self.bitmap_words(pyr.mtb, img, k)),
                               exclusion=Bitmap(w, h, layout, self.bitmap_words(pyr.excl, img, k)),
                               median=int(medians[k]), noise_tolerance=self.tol))
        return out

    # --------------------------------------------------------------- search --
    def maps_table(self, pyr: PyramidSet, pairs) -> "object":
        """Device table [n][P][4] of level pointers {ref.mtb, ref.excl, tgt.mtb, tgt.excl}."""
        pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
        key = (int(pyr.mtb.data_ptr()), int(pyr.excl.data_ptr()), pairs.tobytes())
        tab = self._tables.get(key)
        if tab is not None:
            return tab
        stride = self.bit_img_words * 8
        offs = self.geom[:, 5].astype(np.int64) * 8                                  # [n]
        m0, e0 = int(pyr.mtb.data_ptr()), int(pyr.excl.data_ptr())
        ref, tgt = pairs[:, 0], pairs[:, 1]
        table = np.empty((self.n, len(pairs), 4), dtype=np.int64)
        table[:, :, 0] = m0 + ref[None, :] * stride + offs[:, None]
        table[:, :, 1] = e0 + ref[None, :] * stride + offs[:, None]
        table[:, :, 2] = m0 + tgt[None, :] * stride + offs[:, None]
        table[:, :, 3] = e0 + tgt[None, :] * stride + offs[:, None]
        tab = self.torch.from_numpy(table).to("cuda")
        if len(self._tables) > 64:
            self._tables.clear()
        self._tables[key] = tab
        return tab

    def search_table(self, table, n_pairs: int, acc=None, errs=None, done=None, base=None, count: bool = True):
        """find_offset for every pair of a prepared maps table; results stay on device.

        Returns (acc [P, n, 2] int32 — chosen offset per level, index 0 = full
        resolution; errs [P, n, 9] int64 — candidate errors per level).
        """
        t = self.torch
        if acc is None:
            acc = t.empty((n_pairs, self.n, 2), dtype=t.int32, device="cuda")
        if errs is None:
            errs = t.empty((n_pairs, self.n, 9), dtype=t.int64, device="cuda")
        if done is None:
            done = t.empty((n_pairs, self.n), dtype=t.int32, device="cuda")
        _lib.call("mtb_find_offset_batch", _dev.ptr(table), self.dims.ctypes.data, self.n, n_pairs,
                  _dev.ptr(base) if base is not None else None, _dev.ptr(acc), _dev.ptr(errs), _dev.ptr(done),
                  _dev.stream())
        if count:
            counters.bump(FIND_OFFSET_CALLS, n_pairs)
            counters.bump(SHIFTED_ERROR_EVALS, 9 * self.n * n_pairs)
        return acc, errs

    # ---------------------------------------------------------------- fused --
    @property
    def fused_supported(self) -> bool:
        """True when the one-launch-per-image pipeline (csrc/pipe.cu) handles this geometry."""
        return self.n <= 6 and (3 * self.width) % 16 == 0

    def fused_gray_bytes(self) -> int:
        """Bytes of the fused pipeline's private gray ring (mtb_align_fused_workspace)."""
        gb = getattr(self, "_fused_gray_bytes", None)
        if gb is None:
            arr = np.zeros(1, dtype=np.int64)
            _lib.load().mtb_align_fused_workspace(self.width, self.height, self.requested_levels,
                                                  arr.ctypes.data_as(_lib._i64p), None)
            gb = self._fused_gray_bytes = int(arr[0])
        return gb

    def align_fused(self, rgb, pairs, pyr: PyramidSet | None = None, acc=None, errs=None, done=None,
                    count: bool = True, img_ready=None):
        """Preprocess every image of `rgb` and find_offset every (ref, tgt) pair in ONE
        software-pipelined sequence of launches (csrc/pipe.cu): pipeline.py:80-90
        with search.py:74-95, gray pyramids kept in L2.  Returns (pyr, acc, errs)
        with the same layouts as preprocess + search_table."""
        t = self.torch
        self._check_rgb(rgb)
        if not self.fused_supported:
            raise ValueError("fused path needs <= 6 pyramid levels and 3*W % 16 == 0")
        n_img = int(rgb.shape[0])
        pairs = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
        P = len(pairs)
        if pyr is None:
            pyr = self.alloc(n_img)
        if acc is None:
            acc = t.empty((max(P, 1), self.n, 2), dtype=t.int32, device="cuda")
        if errs is None:
            errs = t.empty((max(P, 1), self.n, 9), dtype=t.int64, device="cuda")
        if done is None:
            done = t.empty((max(P, 1), self.n), dtype=t.int32, device="cuda")
        # Per-call scratch from torch's stream-aware caching allocator (no
        # cudaMalloc after the first call): concurrent calls on different
        # streams never share a gray ring or sync counters.
        gray = t.empty(self.fused_gray_bytes(), dtype=t.uint8, device="cuda")
        words = int(_lib.load().mtb_align_fused_sync_words(n_img, P, self.n))
        sync = t.empty(words, dtype=t.int32, device="cuda")
        _lib.call("mtb_align_fused_ex", _dev.ptr(rgb), 3 * self.width, 3 * self.width * self.height, self.width,
                  self.height, n_img, self.requested_levels, self.tol, pairs.ctypes.data, P, _dev.ptr(gray),
                  _dev.ptr(pyr.hist_ws), _dev.ptr(pyr.medians), _dev.ptr(pyr.mtb), _dev.ptr(pyr.excl),
                  _dev.ptr(acc), _dev.ptr(errs), _dev.ptr(done), _dev.ptr(sync),
                  _dev.ptr(img_ready) if img_ready is not None else None, _dev.stream())
        if count:
            counters.bump(PYRAMID_BUILDS, n_img)
            counters.bump(MTB_PYRAMID_BUILDS, n_img)
            counters.bump(FIND_OFFSET_CALLS, P)
            counters.bump(SHIFTED_ERROR_EVALS, 9 * self.n * P)
        return pyr, acc[:P], errs[:P]

    def fused_launches(self, n_img: int, pairs) -> int:
        """Launch count of align_fused for n_img images and these pairs."""
        pr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
        return int(_lib.load().mtb_align_fused_launches(self.width, self.height, self.requested_levels, int(n_img),
                                                          pr.ctypes.data, len(pr)))

    def align_fused_host(self, host, pairs, pyr: PyramidSet | None = None, acc=None, errs=None, done=None,
                         dev=None, count: bool = True):
        """align_fused on a HOST batch (pinned uint8 [N, H, W, 3], e.g. from
        imageio.load_stack): each image is copied H2D on a side stream and
        flagged with a stream-ordered store; K1 of image i waits for its flag
        inside the pipeline, so the upload overlaps the alignment of the
        images before it.  `dev` is the device batch to fill
        (allocated if None).  Returns (dev, pyr, acc, errs)."""
        t = self.torch
        if host.is_cuda or host.dtype != t.uint8 or host.dim() != 4 or tuple(host.shape[1:]) != (
                self.height, self.width, 3):
            raise ValueError(f"host batch must be a CPU uint8 (N, {self.height}, {self.width}, 3) tensor")
        n_img = int(host.shape[0])
        if dev is None:
            dev = t.empty(tuple(host.shape), dtype=t.uint8, device="cuda")
        cur = t.cuda.current_stream()
        ready = t.empty(max(n_img, 8), dtype=t.int32, device="cuda")   # per call (see align_fused)
        cs = t.cuda.Stream()
        cs.wait_stream(cur)            # dev / ready no longer in use by earlier work
        with t.cuda.stream(cs):
            ready[:n_img].zero_()
        zeroed = t.cuda.Event()
        zeroed.record(cs)
        cur.wait_event(zeroed)         # the pipeline never sees a stale flag
        for i in range(n_img):
            with t.cuda.stream(cs):
                dev[i].copy_(host[i], non_blocking=True)
            _lib.call("mtb_stream_write_u32", _dev.ptr(ready[i]), 1, cs.cuda_stream)
        dev.record_stream(cs)
        ready.record_stream(cs)
        pyr, acc, errs = self.align_fused(dev, pairs, pyr, acc, errs, done, count=count, img_ready=ready)
        cur.wait_stream(cs)
        return dev, pyr, acc, errs

    def search(self, pyr: PyramidSet, pairs, count: bool = True):
        table = self.maps_table(pyr, pairs)
        return self.search_table(table, int(table.shape[1]), count=count)


def results_from_device(acc, errs, base=None) -> list[AlignmentResult]:
    """AlignmentResult per pair (traces deepest first) from the device outputs."""
    acc_h = acc.cpu().numpy()
    errs_h = errs.cpu().numpy()
    out = []
    for p in range(acc_h.shape[0]):
        n = acc_h.shape[1]
        traces = []
        prev = None
        for level in reversed(range(n)):
            if prev is None:
                b = ShiftOffset(0, 0) if base is None else ShiftOffset(int(base[p][0]), int(base[p][1]))
            else:
                b = prev.scaled(2)
            cands = [(ShiftOffset(b.dx + ddx, b.dy + ddy), int(errs_h[p, level, i]))
                     for i, (ddy, ddx) in enumerate(NEIGHBORHOOD)]
            chosen = ShiftOffset(int(acc_h[p, level, 0]), int(acc_h[p, level, 1]))
            traces.append(LevelTrace(level=level, candidates=cands, chosen=chosen, accumulated=chosen))
            prev = chosen
        out.append(AlignmentResult(offset=prev, traces=traces, total_tests=9 * n))
    return out
