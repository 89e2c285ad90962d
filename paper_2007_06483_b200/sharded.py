"""Row-sharded alignment of ONE very large pair over several GPUs
(a 1-gigapixel pair, 10 levels, 8 x B200).

The only configuration whose data path has a real exchange step:

  * rows are split at multiples of 2^(n-1) (n = the pair's level count), so
    every pyramid level partitions exactly and the pyramid needs no halo
    (level-k row y depends on level-0 rows [y*2^k, (y+1)*2^k));
  * each shard builds gray + pyramid + per-level histograms of its rows
    (K1), then the 2 x n x 256 histograms are SUM-all-reduced so every shard
    thresholds with the medians of the whole image (threshold.py:80-88);
  * per level (deepest first) each shard counts the 9 candidate errors over
    its own reference rows; the shifted target rows it needs beyond its own
    (|by|+1 rows, by = the level's base dy) come from the neighbouring shards
    (halo exchange); the 9 counts are SUM-all-reduced and every shard applies
    the same search.py:67 key, so all shards agree on the offset.

Collectives per pair: 1 histogram all-reduce + n x (halo all-gather + one
9-count all-reduce).  `Comm` wraps torch.distributed (NCCL on GPUs, gloo in
the CPU tests); `align_pair_loopback` drives W virtual shards in one process
(same phase functions, sums done in place) for single-GPU verification.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .image import ShiftOffset
from .pyramid import max_levels
from .search import NEIGHBORHOOD, AlignmentResult, LevelTrace


# ------------------------------------------------------------------ geometry --
def plan_row_shards(height: int, n_levels: int, world: int) -> list[tuple[int, int]]:
    """[r0, r1) level-0 row range per shard; r0 multiples of 2^(n-1), the
    remainder rows (< 2^(n-1)) go to the last shard."""
    block = 1 << (n_levels - 1)
    blocks = height // block
    if blocks < world:
        raise ValueError(f"{height} rows make {blocks} blocks of {block}; fewer than {world} shards")
    out, b0 = [], 0
    for r in range(world):
        nb = blocks // world + (1 if r < blocks % world else 0)
        r0, r1 = b0 * block, (b0 + nb) * block
        if r == world - 1:
            r1 = height
        out.append((r0, r1))
        b0 += nb
    return out


def level_rows(r0: int, r1: int, k: int) -> tuple[int, int]:
    return r0 >> k, r1 >> k


def halo_sizes(by: int) -> tuple[int, int]:
    """(rows needed from the previous shard, rows needed from the next shard)
    for output rows searched with base dy = by: source rows y - by + {-1, 0, 1}."""
    return max(0, by + 1), max(0, 1 - by)


# -------------------------------------------------------------- CUDA shard --
class CudaShard:
    """One shard's device state: ref/target rows of one pair and their arenas."""

    def __init__(self, width: int, full_height: int, r0: int, r1: int, n_levels: int, tol: int = 4):
        self.torch = _dev.torch_mod()
        self.w, self.H, self.r0, self.r1, self.n, self.tol = width, full_height, r0, r1, n_levels, tol
        plan = _lib.plan_levels(width, r1 - r0, -n_levels)
        if plan is None:
            raise ValueError(f"shard rows [{r0}, {r1}) cannot hold {n_levels} levels")
        n, self.geom, sizes = plan
        assert n == n_levels
        self.gray_bytes, self.bit_words, self.hist_elems = (int(v) for v in sizes)
        t = self.torch
        self.gray = t.empty((2, self.gray_bytes), dtype=t.uint8, device="cuda")
        self.hist_ws = t.empty((2, self.hist_elems), dtype=t.int32, device="cuda")
        self.mtb = t.empty((2, self.bit_words), dtype=t.int64, device="cuda")
        self.excl = t.empty((2, self.bit_words), dtype=t.int64, device="cuda")
        self.medians = None

    # phase 1: gray + pyramid + local histograms (int64 [2, n, 256])
    def preprocess(self, rgb_rows):
        h = self.r1 - self.r0
        assert tuple(rgb_rows.shape) == (2, h, self.w, 3) and rgb_rows.is_contiguous()
        _lib.call("mtb_pyramid_hist", _dev.ptr(rgb_rows), 3 * self.w, 3 * self.w * h, self.w, h, 2, -self.n,
                  _dev.ptr(self.gray), _dev.ptr(self.hist_ws), _dev.stream())
        spread = self.hist_ws.view(2, -1)[:, : self.n * 256 * 32].view(2, self.n, 256, 32)
        return spread[..., 0].to(self.torch.int64)

    # phase 2: medians of the whole image, threshold + pack own rows
    def threshold(self, global_hist):
        t = self.torch
        med = t.empty(2 * self.n, dtype=t.int32, device="cuda")
        flat = global_hist.reshape(-1, 256).contiguous()
        _lib.call("mtb_median_from_histogram", _dev.ptr(flat), 2 * self.n, _dev.ptr(med), _dev.stream())
        self.medians = med.view(2, self.n)
        _lib.call("mtb_threshold_levels_medians", _dev.ptr(self.gray), self.w, self.r1 - self.r0, 2, -self.n,
                  self.tol, _dev.ptr(med), _dev.ptr(self.mtb), _dev.ptr(self.excl), 0, _dev.stream())

    def level_maps(self, k: int, img: int):
        """(mtb, excl) int64 [rows, nw64] views of level k of image img (0 = ref, 1 = tgt)."""
        h_loc, nw, off = int(self.geom[k, 1]), int(self.geom[k, 4]), int(self.geom[k, 5])
        return (self.mtb[img, off:off + h_loc * nw].view(h_loc, nw),
                self.excl[img, off:off + h_loc * nw].view(h_loc, nw))

    def slabs(self, k: int, hp: int, hn: int):
        """Top hn rows and bottom hp rows of the target maps (both maps stacked)."""
        m, e = self.level_maps(k, 1)
        top = self.torch.stack([m[:hn], e[:hn]])
        bot = self.torch.stack([m[m.shape[0] - hp:], e[e.shape[0] - hp:]])
        return top.contiguous(), bot.contiguous()

    def count_level(self, k: int, lead, tail, prev_dev):
        """9 partial error counts of level k over this shard's reference rows.

        lead: the previous shard's last target rows (2 maps stacked) or None;
        tail: the next shard's first target rows, or None (the halo)."""
        t = self.torch
        am, ae = self.level_maps(k, 0)
        bm, be = self.level_maps(k, 1)
        parts_m = [x for x in (lead[0] if lead is not None else None, bm, tail[0] if tail is not None else None)
                   if x is not None]
        parts_e = [x for x in (lead[1] if lead is not None else None, be, tail[1] if tail is not None else None)
                   if x is not None]
        ext_m, ext_e = t.cat(parts_m).contiguous(), t.cat(parts_e).contiguous()
        y0, y1 = level_rows(self.r0, self.r1, k)
        b_row0 = y0 - (lead.shape[1] if lead is not None else 0)
        w_k, nw = int(self.geom[k, 0]), int(self.geom[k, 4])
        table = t.tensor([[am.data_ptr(), ae.data_ptr(), ext_m.data_ptr(), ext_e.data_ptr()]], dtype=t.int64,
                         device="cuda")
        errs = t.empty((1, 9), dtype=t.int64, device="cuda")
        _lib.call("mtb_search_level_rows", _dev.ptr(table), w_k, self.H >> k, nw, y0, y1 - y0, b_row0,
                  int(ext_m.shape[0]), 1, _dev.ptr(prev_dev) if prev_dev is not None else None, 2,
                  None, _dev.ptr(errs), 9, _dev.stream())
        self._keep = (ext_m, ext_e, table)  # alive until the stream has consumed them
        return errs

    def decide(self, errs_sum, prev_dev):
        """Device decision (search.py:67) from summed counts; returns acc (1, 2) int32."""
        t = self.torch
        acc = t.empty((1, 2), dtype=t.int32, device="cuda")
        _lib.call("mtb_decide_level", _dev.ptr(errs_sum), 9, _dev.ptr(prev_dev) if prev_dev is not None else None,
                  2, None, _dev.ptr(acc), 2, 1, _dev.stream())
        return acc

    def stack_rows(self, ref_rows, tgt_rows):
        return self.torch.stack([_dev.to_device(ref_rows), _dev.to_device(tgt_rows)]).contiguous()


def _result(accs, errs_all, n):
    traces, prev = [], None
    for level in reversed(range(n)):
        b = ShiftOffset(0, 0) if prev is None else prev.scaled(2)
        cands = [(ShiftOffset(b.dx + ddx, b.dy + ddy), int(errs_all[level][i]))
                 for i, (ddy, ddx) in enumerate(NEIGHBORHOOD)]
        chosen = ShiftOffset(int(accs[level][0]), int(accs[level][1]))
        traces.append(LevelTrace(level=level, candidates=cands, chosen=chosen, accumulated=chosen))
        prev = chosen
    return AlignmentResult(offset=prev, traces=traces, total_tests=9 * n)


def pair_levels(width: int, height: int, levels: int) -> int:
    n = min(levels, max_levels(width, height))
    if n < 1:
        raise ValueError(f"images must be at least 16x16; got {width}x{height}")
    return n


# ------------------------------------------------------- loopback driver --
def align_pair_loopback(ref_rgb, tgt_rgb, world: int, levels: int = 10, tol: int = 4,
                        shard_cls=CudaShard) -> AlignmentResult:
    """Row-sharded find_offset of one pair with `world` virtual shards in ONE
    process: the same per-shard phases as the NCCL path, the collectives
    replaced by in-process sums / slab hand-offs.  Bit-identical to the
    unsharded path (tests/test_gpu_sharded.py)."""
    H, W = int(ref_rgb.shape[0]), int(ref_rgb.shape[1])
    n = pair_levels(W, H, levels)
    rows = plan_row_shards(H, n, world)
    shards = [shard_cls(W, H, r0, r1, n, tol) for r0, r1 in rows]
    hists = [sh.preprocess(sh.stack_rows(ref_rgb[r0:r1], tgt_rgb[r0:r1])) for sh, (r0, r1) in zip(shards, rows)]
    ghist = sum(hists[1:], hists[0])
    for sh in shards:
        sh.threshold(ghist)
    prev, accs, errs_all = None, [None] * n, [None] * n
    for k in reversed(range(n)):
        by = 0 if prev is None else 2 * int(prev[0, 1])
        hp, hn = halo_sizes(by)
        sl = [sh.slabs(k, hp, hn) for sh in shards]
        parts = []
        for r, sh in enumerate(shards):
            lead = sl[r - 1][1] if r > 0 and hp > 0 else None
            tail = sl[r + 1][0] if r + 1 < world and hn > 0 else None
            parts.append(sh.count_level(k, lead, tail, prev))
        total = sum(parts[1:], parts[0])
        acc = shards[0].decide(total, prev)
        accs[k], errs_all[k] = np.asarray(acc[0].tolist()), np.asarray(total[0].tolist())
        prev = acc
    return _result(accs, errs_all, n)


# ------------------------------------------------------------- NCCL driver --
def align_pair_distributed(ref_rows, tgt_rows, width: int, height: int, levels: int = 10, tol: int = 4,
                           shard_cls=CudaShard) -> AlignmentResult:
    """SPMD: call on every rank of an initialised torch.distributed group with
    this rank's rows (plan_row_shards(height, n, world)[rank]) of both images.
    NCCL on GPUs (CudaShard); gloo with a CPU shard class in the tests.
    Returns the same AlignmentResult on every rank."""
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    n = pair_levels(width, height, levels)
    r0, r1 = plan_row_shards(height, n, world)[rank]
    shard = shard_cls(width, height, r0, r1, n, tol)
    hist = shard.preprocess(shard.stack_rows(ref_rows, tgt_rows))
    dist.all_reduce(hist, op=dist.ReduceOp.SUM)                   # 2 x n x 256 histograms
    shard.threshold(hist)
    prev, accs, errs_all = None, [None] * n, [None] * n
    for k in reversed(range(n)):
        by = 0 if prev is None else 2 * int(prev[0, 1])
        hp, hn = halo_sizes(by)
        top, bot = shard.slabs(k, hp, hn)
        tops = [top.new_empty(top.shape) for _ in range(world)]
        bots = [bot.new_empty(bot.shape) for _ in range(world)]
        dist.all_gather(tops, top)                                 # halo exchange
        dist.all_gather(bots, bot)
        lead = bots[rank - 1] if rank > 0 and hp > 0 else None
        tail = tops[rank + 1] if rank + 1 < world and hn > 0 else None
        errs = shard.count_level(k, lead, tail, prev)
        dist.all_reduce(errs, op=dist.ReduceOp.SUM)               # 9 counts
        acc = shard.decide(errs, prev)
        accs[k], errs_all[k] = np.asarray(acc[0].tolist()), np.asarray(errs[0].tolist())
        prev = acc
    return _result(accs, errs_all, n)
