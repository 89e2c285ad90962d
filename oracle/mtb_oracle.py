"""CPU ORACLE for the MTB alignment hot path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (mtbalign 0.1.0,
/root/reference/pkg/src/mtbalign).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module, and
only as the checker — the product path (paper_2007_06483_b200) never does.

Pinned: tests/test_oracle_golden.py checks every function here against
golden vectors produced by the UNMODIFIED reference (tests/golden/, made by
tests/golden/make_golden.py from oracle/_ref) and against the reference
tests' own known answers.

Everything is integer arithmetic; results are bit-exact by construction.
The error test is restated on boolean rasters (the reference test oracle's
formulation, tests/conftest.py:14-24) rather than on packed words, so it
shares no shift/popcount code with either engine.
"""

from __future__ import annotations

import numpy as np

MIN_LEVEL_SIZE = 16                       # pyramid.py:14
NEIGHBORHOOD = tuple((ddy, ddx) for ddy in (-1, 0, 1) for ddx in (-1, 0, 1))   # search.py:23


# ---------------------------------------------------------------- image --
def gray(rgb: np.ndarray) -> np.ndarray:
    """image.py:58-68: (54 R + 183 G + 19 B) >> 8, exact in 32-bit ints."""
    c = rgb.astype(np.uint32)
    return ((54 * c[..., 0] + 183 * c[..., 1] + 19 * c[..., 2]) >> 8).astype(np.uint8)


def shift_raster(img: np.ndarray, dx: int, dy: int, fill) -> np.ndarray:
    """image.py:71-106: out(x, y) = img(x - dx, y - dy) in bounds, else fill."""
    h, w = img.shape[:2]
    out = np.empty_like(img)
    out[...] = np.asarray(fill, dtype=img.dtype)
    ys = np.arange(h) - dy
    xs = np.arange(w) - dx
    vy = (ys >= 0) & (ys < h)
    vx = (xs >= 0) & (xs < w)
    if vy.any() and vx.any():
        out[np.ix_(np.flatnonzero(vy), np.flatnonzero(vx))] = img[np.ix_(ys[vy], xs[vx])]
    return out


# -------------------------------------------------------------- pyramid --
def downsample(g: np.ndarray) -> np.ndarray:
    """pyramid.py:17-32: (2x2 sum + 2) >> 2, floor-halved dims."""
    h2, w2 = g.shape[0] // 2, g.shape[1] // 2
    s = g[:2 * h2, :2 * w2].astype(np.uint32).reshape(h2, 2, w2, 2).sum(axis=(1, 3))
    return ((s + 2) >> 2).astype(np.uint8)


def max_levels(w: int, h: int) -> int:
    """pyramid.py:35-42."""
    n = 0
    while w >= MIN_LEVEL_SIZE and h >= MIN_LEVEL_SIZE:
        n, w, h = n + 1, w // 2, h // 2
    return n


def pyramid(g: np.ndarray, levels: int) -> list:
    """pyramid.py:45-62 (no validation; callers pass valid sizes)."""
    n = min(levels, max_levels(g.shape[1], g.shape[0]))
    out = [g]
    for _ in range(n - 1):
        out.append(downsample(out[-1]))
    return out


# ------------------------------------------------------------ threshold --
def histogram(g: np.ndarray) -> np.ndarray:
    """threshold.py:25-28."""
    return np.bincount(g.ravel(), minlength=256).astype(np.int64)


def median(hist: np.ndarray) -> int:
    """threshold.py:31-39: smallest m with cumsum[m] >= (total + 1) // 2."""
    total = int(hist.sum())
    if total < 1:
        raise ValueError("empty histogram")
    target = (total + 1) // 2
    return int(np.argmax(np.cumsum(hist) >= target))


def mtb_mask(g: np.ndarray, med: int) -> np.ndarray:
    """threshold.py:42-45."""
    return g > med


def exclusion_mask(g: np.ndarray, med: int, tol: int) -> np.ndarray:
    """threshold.py:48-56, widened so nothing wraps."""
    return np.abs(g.astype(np.int32) - int(med)) > tol


def pack(mask: np.ndarray) -> np.ndarray:
    """bitmap.py:32-40: LSB-first u64 words, ceil(W/64) per row, zero padding."""
    h, w = mask.shape
    nw = (w + 63) // 64
    bits = np.zeros((h, nw * 64), dtype=np.uint8)
    bits[:, :w] = mask
    weights = (1 << np.arange(64, dtype=np.uint64)).astype(np.uint64)
    return (bits.reshape(h, nw, 64).astype(np.uint64) * weights).sum(axis=2, dtype=np.uint64)


def unpack(words: np.ndarray, w: int) -> np.ndarray:
    h, nw = words.shape
    sh = np.arange(64, dtype=np.uint64)
    bits = (words[:, :, None] >> sh) & np.uint64(1)
    return bits.reshape(h, nw * 64)[:, :w].astype(bool)


def mtb_level(g: np.ndarray, tol: int) -> dict:
    """threshold.py:69-77: one level's median and boolean MTB / exclusion."""
    med = median(histogram(g))
    return {"median": med, "mtb": mtb_mask(g, med), "excl": exclusion_mask(g, med, tol)}


def mtb_pyramid(levels: list, tol: int) -> list:
    """threshold.py:80-88."""
    return [mtb_level(g, tol) for g in levels]


# --------------------------------------------------------------- search --
def shifted_error(a, ea, b, eb, dx: int, dy: int) -> int:
    """conftest.py:14-24 / bitmap.py:102-123 on boolean rasters: count pixels
    (x, y) with 0 <= x-dx < w, 0 <= y-dy < h, a != b(x-dx, y-dy), ea, eb(..)."""
    h, w = a.shape
    x0, x1 = max(dx, 0), w + min(dx, 0)
    y0, y1 = max(dy, 0), h + min(dy, 0)
    if x1 <= x0 or y1 <= y0:
        return 0
    sa = a[y0:y1, x0:x1]
    sb = b[y0 - dy:y1 - dy, x0 - dx:x1 - dx]
    m = (sa != sb) & ea[y0:y1, x0:x1] & eb[y0 - dy:y1 - dy, x0 - dx:x1 - dx]
    return int(np.count_nonzero(m))


def search_level(ref: dict, tgt: dict, base) -> tuple:
    """search.py:53-71: 9 candidates, key (err, |ddx|+|ddy|, index)."""
    bx, by = int(base[0]), int(base[1])
    cands, best, best_key = [], None, None
    for idx, (ddy, ddx) in enumerate(NEIGHBORHOOD):
        off = (bx + ddx, by + ddy)
        err = shifted_error(ref["mtb"], ref["excl"], tgt["mtb"], tgt["excl"], *off)
        cands.append((off, err))
        key = (err, abs(ddx) + abs(ddy), idx)
        if best_key is None or key < best_key:
            best_key, best = key, off
    return best, cands


def find_offset(ref_levels: list, tgt_levels: list) -> dict:
    """search.py:74-95: deepest first, base = 2 * accumulated."""
    acc = (0, 0)
    traces = []
    for level in reversed(range(len(ref_levels))):
        base = (2 * acc[0], 2 * acc[1])
        chosen, cands = search_level(ref_levels[level], tgt_levels[level], base)
        acc = chosen
        traces.append({"level": level, "candidates": cands, "chosen": chosen})
    return {"offset": acc, "traces": traces, "total_tests": 9 * len(ref_levels)}


def brute_force(ref: dict, tgt: dict, radius: int) -> tuple:
    """search.py:98-119."""
    best, best_key, idx = None, None, 0
    for dy in range(-radius, radius + 1):
        for dx in range(-radius, radius + 1):
            err = shifted_error(ref["mtb"], ref["excl"], tgt["mtb"], tgt["excl"], dx, dy)
            key = (err, abs(dx) + abs(dy), idx)
            if best_key is None or key < best_key:
                best_key, best = key, ((dx, dy), err)
            idx += 1
    return best


# ------------------------------------------------------------- pipeline --
def preprocess(rgb: np.ndarray, levels: int = 6, tol: int = 4) -> dict:
    """pipeline.py:80-85 for one image: gray, pyramid, MTB pyramid."""
    g = gray(rgb)
    pyr = pyramid(g, levels)
    return {"gray": g, "pyramid": pyr, "mtb": mtb_pyramid(pyr, tol)}


def align_pairs(images: list, pairs: list, levels: int = 6, tol: int = 4) -> list:
    """find_offset over (ref, tgt) index pairs, each image preprocessed once."""
    pre = [preprocess(im, levels, tol) for im in images]
    return [find_offset(pre[r]["mtb"], pre[t]["mtb"]) for r, t in pairs]


def align_stack(images: list, levels: int = 6, tol: int = 4) -> tuple:
    """pipeline.py:52-120: chain pairs, prefix-summed offsets, shifted outputs."""
    results = align_pairs(images, [(i, i + 1) for i in range(len(images) - 1)], levels, tol)
    cum = [(0, 0)]
    for r in results:
        cum.append((cum[-1][0] + r["offset"][0], cum[-1][1] + r["offset"][1]))
    aligned = [images[0]] + [shift_raster(im, c[0], c[1], (0, 0, 0)) for im, c in zip(images[1:], cum[1:])]
    return aligned, results, cum


def align_pivot(images: list, pivot: int, levels: int = 6, tol: int = 4) -> tuple:
    """Pivot pairing (config 3): find_offset(mtb[pivot], mtb[i]) for every i."""
    others = [i for i in range(len(images)) if i != pivot]
    results = align_pairs(images, [(pivot, i) for i in others], levels, tol)
    cum = [(0, 0)] * len(images)
    for i, r in zip(others, results):
        cum[i] = r["offset"]
    aligned = [im if i == pivot else shift_raster(im, cum[i][0], cum[i][1], (0, 0, 0))
               for i, im in enumerate(images)]
    return aligned, results, cum


# ---------------------------------------------------------- input recipes --
def tone_lut(gain: float, gamma: float) -> np.ndarray:
    """synth.py:25-29."""
    v = np.arange(256, dtype=np.float64) / 255.0
    return np.clip(np.round(255.0 * np.power(gain * v, 1.0 / gamma)), 0, 255).astype(np.uint8)


def generate_stack(base: np.ndarray, count: int, pairwise=None, seed: int = 0, max_shift: int = 16,
                   gains=None, gammas=None) -> tuple:
    """synth.py:45-103 (same Generator draw order: offsets, gains, gammas)."""
    rng = np.random.default_rng(seed)
    if pairwise is None:
        pairwise = [(int(rng.integers(-max_shift, max_shift + 1)), int(rng.integers(-max_shift, max_shift + 1)))
                    for _ in range(count - 1)]
    if gains is None:
        gains = [float(rng.uniform(0.5, 2.0)) for _ in range(count)]
    if gammas is None:
        gammas = [float(rng.uniform(0.7, 1.4)) for _ in range(count)]
    cum = [(0, 0)]
    for o in pairwise:
        cum.append((cum[-1][0] + int(o[0]), cum[-1][1] + int(o[1])))
    imgs = []
    for i in range(count):
        disp = shift_raster(base, -cum[i][0], -cum[i][1], (0, 0, 0)) if i else base
        imgs.append(tone_lut(gains[i], gammas[i])[disp])
    return imgs, {"pairwise": [list(map(int, o)) for o in pairwise], "cumulative": [list(c) for c in cum],
                  "gains": gains, "gammas": gammas}


def smooth_gray(rng, w: int, h: int, cells: int = 8, detail: float = 12.0) -> np.ndarray:
    """tests/conftest.py:56-77 (bilinear-upscaled coarse noise plus detail)."""
    small = rng.uniform(0, 255, size=(cells, cells))
    ys = np.linspace(0, cells - 1, h)
    xs = np.linspace(0, cells - 1, w)
    y0 = np.floor(ys).astype(int)
    x0 = np.floor(xs).astype(int)
    y1 = np.minimum(y0 + 1, cells - 1)
    x1 = np.minimum(x0 + 1, cells - 1)
    fy = (ys - y0)[:, None]
    fx = (xs - x0)[None, :]
    up = (small[np.ix_(y0, x0)] * (1 - fy) * (1 - fx) + small[np.ix_(y0, x1)] * (1 - fy) * fx
          + small[np.ix_(y1, x0)] * fy * (1 - fx) + small[np.ix_(y1, x1)] * fy * fx)
    out = up + rng.normal(0, detail, size=(h, w))
    return np.clip(np.round(out), 0, 255).astype(np.uint8)


def synthetic_gray(rng, w: int, h: int, cells: int = 12) -> np.ndarray:
    """benchmarks/engine_bench.py:22-35."""
    ys = np.linspace(0, cells - 1, h)
    xs = np.linspace(0, cells - 1, w)
    coarse = rng.uniform(0, 255, size=(cells, cells))
    iy = np.clip(ys.astype(int), 0, cells - 2)
    ix = np.clip(xs.astype(int), 0, cells - 2)
    fy = (ys - iy)[:, None]
    fx = (xs - ix)[None, :]
    img = (coarse[np.ix_(iy, ix)] * (1 - fy) * (1 - fx) + coarse[np.ix_(iy, ix + 1)] * (1 - fy) * fx
           + coarse[np.ix_(iy + 1, ix)] * fy * (1 - fx) + coarse[np.ix_(iy + 1, ix + 1)] * fy * fx)
    img += rng.normal(0, 10, size=(h, w))
    return np.clip(np.round(img), 0, 255).astype(np.uint8)
