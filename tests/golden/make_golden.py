#!/usr/bin/env python3
"""Generate golden vectors from the UNMODIFIED reference (mtbalign 0.1.0).

Run in the build container, where the reference is built into oracle/_ref by
oracle/build_ref.sh:

    python tests/golden/make_golden.py

Writes tests/golden/golden.npz (arrays) and tests/golden/golden.json
(scalars, traces, input checksums).  Inputs are either stored (small) or
regenerated in the tests from the recorded seeds with the oracle's copies of
the reference recipes; their sha256 is recorded so a recipe drift fails
loudly.  The reference is used through its public API with its compiled
(Cython) engine, and every error count is cross-checked against its numpy
engine too.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import mtbalign as ref  # noqa: E402  (the reference package)
from mtbalign import kernels as ref_kernels  # noqa: E402
from mtbalign.kernels import fallback as ref_fallback  # noqa: E402

import mtb_oracle as orc  # noqa: E402  (only for the shared input recipes)

assert ref_kernels.engine_name() == "native", "build oracle/_ref first (oracle/build_ref.sh)"
_native = ref_kernels.active()


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


arrays: dict = {}
meta: dict = {"reference": "mtbalign " + ref.__version__, "engine": ref_kernels.engine_name()}


def put(name, arr):
    arrays[name] = np.ascontiguousarray(arr)
    return name


# -- A. grayscale (test_image.py recipe) ----------------------------------
rs = np.random.RandomState(7)
rgb = rs.randint(0, 256, size=(13, 9, 3), dtype=np.uint8)
put("gray_in", rgb)
put("gray_out", ref.to_grayscale(rgb))
solid = np.array([[[255, 0, 0], [0, 0, 0], [255, 255, 255], [1, 2, 3]]], dtype=np.uint8)
put("gray_solid_in", solid)
put("gray_solid_out", ref.to_grayscale(solid))

# -- B. pyramids, histograms, medians, bitmaps -----------------------------
pyr_cases = []
rs = np.random.RandomState(44)
for ci, (h, w, L, tol) in enumerate([(130, 90, 4, 4), (77, 53, 3, 4), (64, 64, 6, 4), (100, 129, 6, 0),
                                     (33, 47, 2, 7), (16, 16, 3, 4), (97, 200, 5, 4)]):
    img = rs.randint(0, 256, size=(h, w), dtype=np.uint8)
    if ci == 3:  # saturated masses at 0 and 255 (gain-2 exposure style)
        img = np.clip(img.astype(np.int32) * 2 - 128, 0, 255).astype(np.uint8)
    put(f"pyr{ci}_in", img)
    levels = ref.build_pyramid(img, L)
    pairs = ref.build_mtb_pyramid(levels, tol)
    rec = {"h": h, "w": w, "levels_requested": L, "tol": tol, "n": len(levels), "medians": []}
    for k, (lv, pr) in enumerate(zip(levels, pairs)):
        put(f"pyr{ci}_l{k}", lv)
        put(f"pyr{ci}_h{k}", ref.histogram(lv))
        put(f"pyr{ci}_m{k}", pr.mtb.buf)
        put(f"pyr{ci}_e{k}", pr.exclusion.buf)
        rec["medians"].append(pr.median)
    pyr_cases.append(rec)
meta["pyramid_cases"] = pyr_cases

# -- C. packed shifted error (test_kernels.py:60-82 recipe) ----------------
shift_cases = []
rs = np.random.RandomState(31)
for i in range(60):
    w, h = int(rs.randint(1, 150)), int(rs.randint(1, 25))
    masks = [(rs.rand(h, w) < rs.rand()) for _ in range(4)]
    dx = int(rs.randint(-w - 70, w + 71))
    dy = int(rs.randint(-h - 3, h + 4))
    packed = [ref.Bitmap.from_bool(m, "packed").buf for m in masks]
    e = _native.shifted_error_packed(*packed, dx, dy)
    assert e == ref_fallback.shifted_error_packed(*packed, dx, dy)
    for j, p in enumerate(packed):
        put(f"se{i}_{j}", p)
    shift_cases.append({"w": w, "h": h, "dx": dx, "dy": dy, "err": int(e)})
rs = np.random.RandomState(32)
masks = [(rs.rand(9, 200) < 0.5) for _ in range(4)]
packed = [ref.Bitmap.from_bool(m, "packed").buf for m in masks]
for j, p in enumerate(packed):
    put(f"wb_{j}", p)
wb = []
for dx in (-200, -129, -128, -127, -65, -64, -63, -33, -32, -31, -1, 0, 1, 31, 32, 33, 63, 64, 65, 127, 128,
           129, 200):
    for dy in (-1, 0, 2):
        e = _native.shifted_error_packed(*packed, dx, dy)
        assert e == ref_fallback.shifted_error_packed(*packed, dx, dy)
        wb.append({"dx": dx, "dy": dy, "err": int(e)})
meta["shift_cases"] = shift_cases
meta["word_boundary"] = {"w": 200, "h": 9, "cases": wb}
# count_ones
rs = np.random.RandomState(30)
cnt = []
for i in range(20):
    w, h = int(rs.randint(1, 200)), int(rs.randint(1, 30))
    b = ref.Bitmap.from_bool(rs.rand(h, w) < 0.5, "packed")
    put(f"co{i}", b.buf)
    cnt.append({"w": w, "h": h, "count": int(b.count_ones())})
meta["count_cases"] = cnt


# -- D. find_offset traces (test_search.py displaced_pyramid recipe) -------
def trace_json(res):
    return {"offset": list(res.offset), "total_tests": res.total_tests,
            "traces": [{"level": t.level, "chosen": list(t.chosen), "accumulated": list(t.accumulated),
                        "candidates": [[o.dx, o.dy, int(e)] for o, e in t.candidates]} for t in res.traces]}


search_cases = []
for seed, (w, h), disp, L in [(66, (200, 160), (-5, 3), 4), (70, (128, 128), (-3, 2), 3), (62, (40, 30), (-1, 0), 1),
                              (69, (72, 60), (2, 2), 2), (101, (257, 190), (13, -9), 5), (102, (300, 221), (-30, 17), 6)]:
    rng = np.random.default_rng(seed)
    g = orc.smooth_gray(rng, w, h)
    med = ref.median_from_histogram(ref.histogram(g))
    moved = ref.shift_gray(g, ref.ShiftOffset(*disp), fill=med)
    rp = ref.build_mtb_pyramid(ref.build_pyramid(g, L))
    tp = ref.build_mtb_pyramid(ref.build_pyramid(moved, L))
    res = ref.find_offset(rp, tp)
    put(f"srch_ref_{seed}", g)
    put(f"srch_tgt_{seed}", moved)
    rec = {"seed": seed, "w": w, "h": h, "disp": list(disp), "levels": L, "result": trace_json(res)}
    bf_off, bf_err = ref.brute_force_offset(rp[0], tp[0], 3)
    rec["brute3"] = [bf_off.dx, bf_off.dy, int(bf_err)]
    search_cases.append(rec)
meta["search_cases"] = search_cases

# -- E. align_stack on generated stacks (test_pipeline.py recipe) ----------
stack_cases = []
for seed, (w, h), pairwise in [(84, (256, 256), [(3, 2), (-1, 4)]), (87, (200, 160), [(4, -2), (-3, 5)]),
                               (83, (256, 256), [(1, 0), (2, 1)])]:
    rng = np.random.default_rng(seed)
    base = np.dstack([orc.smooth_gray(rng, w, h) for _ in range(3)])
    gseed = int(rng.integers(2 ** 31))
    images, manifest = ref.generate_stack(base, len(pairwise) + 1, pairwise=[ref.ShiftOffset(*p) for p in pairwise],
                                          seed=gseed)
    aligned, record = ref.align_stack(images)
    stack_cases.append({
        "seed": seed, "w": w, "h": h, "pairwise_in": pairwise, "gen_seed": gseed,
        "input_sha": [sha(im) for im in images], "manifest": manifest,
        "cumulative": [list(c) for c in record.cumulative],
        "pairwise": [trace_json(r) for r in record.pairwise],
        "aligned_sha": [sha(a) for a in aligned],
    })
meta["stack_cases"] = stack_cases

# -- F. config 1: 1024x768 pairs, 6 levels, shifts up to +-63 --------------
cfg1 = []
rng = np.random.default_rng(0)
ga = orc.synthetic_gray(rng, 1024, 768)
gb = orc.synthetic_gray(rng, 1024, 768)
gc = orc.synthetic_gray(rng, 1024, 768)
base = np.dstack([ga, gb, gc])
meta["cfg1_base_sha"] = sha(base)
fixed = [None, [(0, 0)], [(1, 0)], [(-5, 3)], [(63, -63)], [(-63, 63)], [(64, 0)], [(-64, 10)]]
for s in range(8):
    pw = fixed[s] if s < len(fixed) else None
    images, manifest = ref.generate_stack(base, 2, pairwise=pw, seed=s, max_shift=63)
    aligned, record = ref.align_stack(images)
    cfg1.append({"seed": s, "pairwise_in": pw, "input_sha": [sha(im) for im in images],
                 "manifest_pairwise": manifest["pairwise"], "offset": list(record.cumulative[1]),
                 "result": trace_json(record.pairwise[0]), "aligned_sha": sha(aligned[1]),
                 "medians": [p.median for p in ref.build_mtb_pyramid(ref.build_pyramid(ref.to_grayscale(images[1]), 6))]})
meta["cfg1"] = cfg1

# degenerate images (test_search.py:65-72): constant and all-255
deg = []
for val in (100, 255, 0):
    img = np.full((96, 128, 3), val, dtype=np.uint8)
    aligned, record = ref.align_stack([img, img.copy()])
    deg.append({"value": val, "offset": list(record.cumulative[1]), "result": trace_json(record.pairwise[0])})
meta["degenerate"] = deg

out_dir = os.path.dirname(os.path.abspath(__file__))
np.savez_compressed(os.path.join(out_dir, "golden.npz"), **arrays)
with open(os.path.join(out_dir, "golden.json"), "w") as f:
    json.dump(meta, f, indent=1)
print("wrote", len(arrays), "arrays;", os.path.getsize(os.path.join(out_dir, "golden.npz")), "bytes npz")
