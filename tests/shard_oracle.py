"""CPU stand-in for CudaShard (test infrastructure): the same per-shard
phases computed with the numpy oracle, so the row-sharded orchestration
(histogram all-reduce, neighbour halo exchange, 9-count all-reduce) can be exercised
with gloo on CPU."""

import numpy as np
import torch

import mtb_oracle as orc
from paper_2007_06483_b200.sharded import level_rows


class OracleShard:
    def __init__(self, width, full_height, r0, r1, n_levels, tol=4):
        self.w, self.H, self.r0, self.r1, self.n, self.tol = width, full_height, r0, r1, n_levels, tol

    def stack_rows(self, ref_rows, tgt_rows):
        return np.stack([np.asarray(ref_rows), np.asarray(tgt_rows)])

    def preprocess(self, rgb_rows):
        self.levels = []
        hist = np.zeros((2, self.n, 256), np.int64)
        for i in range(2):
            g = orc.gray(rgb_rows[i])
            lv = [g]
            for _ in range(self.n - 1):
                lv.append(orc.downsample(lv[-1]))
            self.levels.append(lv)
            for k in range(self.n):
                hist[i, k] = orc.histogram(lv[k])
        return torch.from_numpy(hist)

    def threshold(self, global_hist):
        gh = global_hist.numpy()
        self.maps = [[None] * self.n for _ in range(2)]
        for i in range(2):
            for k in range(self.n):
                med = orc.median(gh[i, k])
                g = self.levels[i][k]
                self.maps[i][k] = (orc.mtb_mask(g, med).astype(np.uint8),
                                   orc.exclusion_mask(g, med, self.tol).astype(np.uint8))

    def edges(self, k, rows):
        m, e = self.maps[1][k]
        return ((torch.from_numpy(m[:rows].copy()), torch.from_numpy(e[:rows].copy())),
                (torch.from_numpy(m[m.shape[0] - rows:].copy()), torch.from_numpy(e[e.shape[0] - rows:].copy())))

    def halo_buffers(self, k, rows):
        w = self.maps[1][k][0].shape[1]
        return torch.empty((rows, w), dtype=torch.uint8), torch.empty((rows, w), dtype=torch.uint8)

    def count_level(self, k, lead, tail, prev, halo):
        am, ae = self.maps[0][k]
        bm, be = self.maps[1][k]
        parts_m = [p for p in (lead[0].numpy() if lead is not None else None, bm,
                               tail[0].numpy() if tail is not None else None) if p is not None]
        parts_e = [p for p in (lead[1].numpy() if lead is not None else None, be,
                               tail[1].numpy() if tail is not None else None) if p is not None]
        ext_m, ext_e = np.concatenate(parts_m), np.concatenate(parts_e)
        y0, y1 = level_rows(self.r0, self.r1, k)
        b0 = y0 - (halo if lead is not None else 0)
        hk, wk = self.H >> k, am.shape[1]
        bx, by = (0, 0) if prev is None else (2 * int(prev[0, 0]), 2 * int(prev[0, 1]))
        errs = np.zeros(9, np.int64)
        for idx, (ddy, ddx) in enumerate(orc.NEIGHBORHOOD):
            dx, dy = bx + ddx, by + ddy
            total = 0
            for y in range(y0, y1):
                sy = y - dy
                if not (0 <= sy < hk and b0 <= sy < b0 + ext_m.shape[0]):
                    continue
                a, ea = am[y - y0].astype(bool), ae[y - y0].astype(bool)
                b, eb = ext_m[sy - b0].astype(bool), ext_e[sy - b0].astype(bool)
                x0, x1 = max(dx, 0), wk + min(dx, 0)
                if x1 > x0:
                    total += int(np.count_nonzero((a[x0:x1] != b[x0 - dx:x1 - dx]) & ea[x0:x1] & eb[x0 - dx:x1 - dx]))
            errs[idx] = total
        return torch.from_numpy(errs[None])

    def decide(self, errs_sum, prev):
        bx, by = (0, 0) if prev is None else (2 * int(prev[0, 0]), 2 * int(prev[0, 1]))
        e = errs_sum[0].tolist()
        best = min(range(9), key=lambda i: (e[i], abs(i % 3 - 1) + abs(i // 3 - 1), i))
        return torch.tensor([[bx + best % 3 - 1, by + best // 3 - 1]], dtype=torch.int32)
