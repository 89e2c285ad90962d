"""Row-sharded alignment of ONE very large pair over several GPUs
(a 1-gigapixel pair, 10 levels, 8 x B200).

The only configuration whose data path has a real exchange step:

  * rows are split at multiples of 2^(n-1) (n = the pair's level count), so
    every pyramid level partitions exactly and the pyramid needs no halo
    (level-k row y depends on level-0 rows [y*2^k, (y+1)*2^k));
  * each shard builds gray + pyramid + per-level histograms of its rows
    (K1), then the 2 x n x 256 histograms are SUM-all-reduced so every shard
    thresholds with the medians of the whole image (threshold.py:80-88);
  * the shifted target rows a shard needs beyond its own come from its two
    neighbours only: at level k the base dy is 2 * acc(k+1) with
    |acc(j)| <= 2^(n-j) - 1, so the candidates read at most 2^(n-k) - 1 rows
    past either edge (`halo_rows`).  Shards hold >= 2 blocks of 2^(n-1) rows,
    so that halo is always shorter than a neighbour's rows.  These worst-case
    halos of every level are exchanged ONCE per pair, right after the
    threshold pass, in one batched neighbour send/recv (NCCL P2P over
    NVLink); nothing depends on the chosen offsets on the host;
  * per level (deepest first) each shard counts the 9 candidate errors over
    its own reference rows against [previous halo | own rows | next halo]
    (three buffers, mtb_search_level_rows3: no concatenation), the 9 counts
    are SUM-all-reduced and every shard applies the same search.py:67 key on
    the device, so all shards agree on the offset without a host round trip.

Collectives per pair: 1 histogram all-reduce + 1 batched halo exchange + n
9-count all-reduces; the level loop has no host synchronisation.
`align_pair_loopback` drives W virtual shards in one process (same phase
functions, sums done in place) for single-GPU verification.
"""

from __future__ import annotations

import ctypes


from . import _dev, _lib
from .image import ShiftOffset
from .pyramid import max_levels
from .search import NEIGHBORHOOD, AlignmentResult, LevelTrace


# ------------------------------------------------------------------ geometry --
def plan_row_shards(height: int, n_levels: int, world: int) -> list[tuple[int, int]]:
    """[r0, r1) level-0 row range per shard; r0 multiples of 2^(n-1), the
    remainder rows (< 2^(n-1)) go to the last shard.  Every shard gets >= 2
    blocks so its neighbours' worst-case halos (`halo_rows`) fit in it."""
    block = 1 << (n_levels - 1)
    blocks = height // block
    if blocks < 2 * world:
        raise ValueError(f"{height} rows make {blocks} blocks of {block}; need >= 2 per shard for {world} shards")
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


def halo_rows(n_levels: int, k: int) -> int:
    """Worst-case target rows needed past either shard edge at level k:
    |base dy| + 1 <= 2 (2^(n-1-k) - 1) + 1 = 2^(n-k) - 1 (search.py:85-95)."""
    return (1 << (n_levels - k)) - 1


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

    def edges(self, k: int, rows: int):
        """((mtb, excl) of the first `rows`, (mtb, excl) of the last `rows`) target
        rows of level k: contiguous views, sent to the neighbours as halos."""
        m, e = self.level_maps(k, 1)
        return (m[:rows], e[:rows]), (m[m.shape[0] - rows:], e[e.shape[0] - rows:])

    def halo_buffers(self, k: int, rows: int):
        nw = int(self.geom[k, 4])
        t = self.torch
        return (t.empty((rows, nw), dtype=t.int64, device="cuda"), t.empty((rows, nw), dtype=t.int64, device="cuda"))

    def count_level(self, k: int, lead, tail, prev_dev, halo: int):
        """9 partial error counts (1, 9) of level k over this shard's reference rows
        against the target window [lead | own | tail]; lead / tail = (mtb, excl)
        halo buffers of `halo` rows from the neighbours, or None at an image edge."""
        t = self.torch
        am, ae = self.level_maps(k, 0)
        bm, be = self.level_maps(k, 1)
        y0, y1 = level_rows(self.r0, self.r1, k)
        w_k, nw = int(self.geom[k, 0]), int(self.geom[k, 4])
        segs = (ctypes.c_void_p * 6)(
            lead[0].data_ptr() if lead is not None else None, lead[1].data_ptr() if lead is not None else None,
            bm.data_ptr(), be.data_ptr(),
            tail[0].data_ptr() if tail is not None else None, tail[1].data_ptr() if tail is not None else None)
        row0 = (ctypes.c_int * 3)(y0 - halo, y0, y1)
        rows = (ctypes.c_int * 3)(halo if lead is not None else 0, y1 - y0, halo if tail is not None else 0)
        errs = t.empty((1, 9), dtype=t.int64, device="cuda")
        _lib.call("mtb_search_level_rows3", am.data_ptr(), ae.data_ptr(), y0, y1 - y0, segs, row0, rows, w_k,
                  self.H >> k, nw, _dev.ptr(prev_dev) if prev_dev is not None else None, None, _dev.ptr(errs),
                  _dev.stream())
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
    replaced by in-process sums and halo hand-offs (neighbour edge views).
    Bit-identical to the unsharded path (tests/test_gpu_sharded.py)."""
    H, W = int(ref_rgb.shape[0]), int(ref_rgb.shape[1])
    n = pair_levels(W, H, levels)
    rows = plan_row_shards(H, n, world)
    shards = [shard_cls(W, H, r0, r1, n, tol) for r0, r1 in rows]
    hists = [sh.preprocess(sh.stack_rows(ref_rgb[r0:r1], tgt_rgb[r0:r1])) for sh, (r0, r1) in zip(shards, rows)]
    ghist = sum(hists[1:], hists[0])
    for sh in shards:
        sh.threshold(ghist)
    accs, errs_all = loopback_levels(shards, n)
    return _result([a[0].tolist() for a in accs], [e[0].tolist() for e in errs_all], n)


def loopback_levels(shards, n: int):
    """The coarse-to-fine level loop over in-process shards; returns the
    per-level device tensors (chosen offset (1, 2), summed counts (1, 9)).
    Issues no synchronising call (tests/test_gpu_sharded.py)."""
    world = len(shards)
    prev, accs, errs_all = None, [None] * n, [None] * n
    for k in reversed(range(n)):
        hk = halo_rows(n, k)
        edges = [sh.edges(k, hk) for sh in shards]
        parts = [sh.count_level(k, edges[r - 1][1] if r > 0 else None, edges[r + 1][0] if r + 1 < world else None,
                                prev, hk) for r, sh in enumerate(shards)]
        total = parts[0]
        for p in parts[1:]:
            total = total + p
        prev = shards[0].decide(total, prev)
        accs[k], errs_all[k] = prev, total
    return accs, errs_all


# ------------------------------------------------------------- NCCL driver --
def exchange_halos(shard, n: int, rank: int, world: int):
    """Every level's worst-case halos in ONE batched neighbour exchange:
    this shard's first rows go to rank-1 (its `tail`), its last rows to rank+1
    (its `lead`).  Returns {k: (lead, tail)} (None at the image edges)."""
    import torch.distributed as dist

    ops, out = [], {}
    for k in range(n):
        hk = halo_rows(n, k)
        top, bot = shard.edges(k, hk)
        lead = shard.halo_buffers(k, hk) if rank > 0 else None
        tail = shard.halo_buffers(k, hk) if rank + 1 < world else None
        if lead is not None:
            ops += [dist.P2POp(dist.isend, top[0], rank - 1), dist.P2POp(dist.isend, top[1], rank - 1),
                    dist.P2POp(dist.irecv, lead[0], rank - 1), dist.P2POp(dist.irecv, lead[1], rank - 1)]
        if tail is not None:
            ops += [dist.P2POp(dist.isend, bot[0], rank + 1), dist.P2POp(dist.isend, bot[1], rank + 1),
                    dist.P2POp(dist.irecv, tail[0], rank + 1), dist.P2POp(dist.irecv, tail[1], rank + 1)]
        out[k] = (lead, tail)
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return out


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
    halos = exchange_halos(shard, n, rank, world)                 # all levels, one batched P2P
    prev, accs, errs_all = None, [None] * n, [None] * n
    for k in reversed(range(n)):                                  # no host synchronisation in here
        lead, tail = halos[k]
        errs = shard.count_level(k, lead, tail, prev, halo_rows(n, k))
        dist.all_reduce(errs, op=dist.ReduceOp.SUM)               # 9 counts
        prev = shard.decide(errs, prev)
        accs[k], errs_all[k] = prev, errs
    return _result([a[0].tolist() for a in accs], [e[0].tolist() for e in errs_all], n)
