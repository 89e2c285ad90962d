#!/usr/bin/env python3
"""Benchmark: aligned pairs/sec at 24 MP RGB8, 6 levels (BASELINE.json metric).

Workload (config 2 of BASELINE.json, made throughput-shaped): every step
aligns `--pairs` independent 6000x4000 RGB8 exposure pairs per GPU with 6
pyramid levels and tol 4 — the full hot path: fused gray + pyramid +
histograms, medians, threshold/pack of every level, and the 6-level
coarse-to-fine search of every pair, all on the device.  Inputs are
synthetic exposure pairs generated on the device before timing (a base scene
and a shifted, tone-mapped second exposure, synth.py recipe) and are larger
than L2 (pairs x 144 MB), so no L2 flush is needed between steps.

Multi-GPU (torchrun): batch-sharding, each rank aligns its own pairs; no
collective on the data path (weak scaling).  Time = max over ranks of the
CUDA-event time of K steps between barriers.

`--impl reference` times the reference's own CPU implementation (oracle/_ref:
mtbalign 0.1.0 with its compiled engine, align_stack on all host cores) on a
bounded sample of the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "aligned pairs/sec at 24MP RGB8, 6 levels; % of B200 HBM roofline"
UNIT = "pairs/s"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, choices=(1, 2, 3, 4), default=2,
                    help="BASELINE.json config: 1 = 1024x768 pairs, 2 = 24 MP pairs (default, the headline), "
                         "3 = 7 x 24 MP stacks aligned to the middle exposure, 4 = 12 MP pairs")
    ap.add_argument("--pairs", type=int, default=0, help="pairs (config 3: stacks) per step per GPU; 0 = config default")
    ap.add_argument("--width", type=int, default=0)
    ap.add_argument("--height", type=int, default=0)
    ap.add_argument("--levels", type=int, default=6)
    ap.add_argument("--tol", type=int, default=4)
    ap.add_argument("--mode", choices=("fused", "staged"), default="fused",
                    help="fused: one pipelined launch per image (csrc/pipe.cu); staged: K1 / K3 / K4 kernels")
    ap.add_argument("--chunk", type=int, default=0,
                    help="images per preprocess round (K1 launches then threshold); 0 = whole batch")
    ap.add_argument("--keep-gray", action="store_true", help="do not discard consumed gray lines from L2")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-graph", action="store_true", help="launch every kernel from Python instead of a CUDA graph")
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-oracle-check", action="store_true", help="skip checking every benched pair on the CPU")
    args = ap.parse_args()
    dflt = CONFIGS[args.config]
    args.width = args.width or dflt["width"]
    args.height = args.height or dflt["height"]
    args.pairs = args.pairs or dflt["units"]
    args.stack = dflt["stack"]
    if "--mode" not in " ".join(sys.argv):
        # the product's own dispatch (pipeline.use_fused)
        args.mode = "fused" if fused_default(args.width, args.height, args.pairs * args.stack) else "staged"
    return args


# BASELINE.json configs as bench workloads: `units` per step per GPU of
# `stack` images each (pairs: stack 2; config 3: 7-exposure stacks aligned to
# their middle exposure, 6 pairs each).  Config 5 (one gigapixel pair,
# row-sharded) is measured by tools/config5.py, not here.
# = paper_2007_06483_b200.pipeline's dispatch tables (checked by tests)
FUSED_MIN_PIXELS = 13_000_000
FUSED_MIN_IMAGES = {20_000_000: 20, FUSED_MIN_PIXELS: 96}


def fused_default(width: int, height: int, n_img: int) -> bool:
    for min_px, min_img in sorted(FUSED_MIN_IMAGES.items(), reverse=True):
        if width * height >= min_px:
            return n_img >= min_img
    return False


CONFIGS = {
    1: {"width": 1024, "height": 768, "units": 1024, "stack": 2},
    2: {"width": 6000, "height": 4000, "units": 64, "stack": 2},
    3: {"width": 6000, "height": 4000, "units": 16, "stack": 7},
    4: {"width": 4000, "height": 3000, "units": 128, "stack": 2},
}


def unit_pairs(n_units: int, stack: int):
    """(ref, tgt) image pairs of n_units stacks of `stack` images: pairs for
    stack 2, else every exposure against the stack's middle one."""
    if stack == 2:
        return [(2 * u, 2 * u + 1) for u in range(n_units)]
    mid = stack // 2
    return [(stack * u + mid, stack * u + i) for u in range(n_units) for i in range(stack) if i != mid]


def load_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(kernel: str, width: int, height: int, images_per_launch: int):
    """Per-launch DRAM bytes of `kernel` at this workload (W x H, images per
    launch) from the committed ncu summary; None when no capture matches."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d["by_workload"].get(f"{kernel}:{width}x{height}x{images_per_launch}")
    except Exception:
        return None


# ------------------------------------------------------------- clocks --
class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self._nv is not None:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------- CPU reference --
def reference_images(width, height, stack=2, seed=1):
    """The bounded CPU sample: one exposure pair (or one 7-exposure config-3
    stack) from the device generator's recipe, built with numpy here."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import mtb_oracle as orc

    rng = np.random.default_rng(seed)
    base = np.dstack([orc.synthetic_gray(rng, width, height) for _ in range(3)])
    if stack == 2:
        return orc.generate_stack(base, 2, seed=seed, max_shift=63)
    return orc.generate_stack(base, stack, seed=seed, max_shift=20, gains=[2 ** ((k - 3) / 3) for k in range(stack)],
                              gammas=[1.0] * stack)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def time_reference(width, height, levels, tol, reps, stack=2):
    """Reference align_stack (oracle/_ref, compiled engine) on all host cores and
    on one worker; pairs/s (a stack of k images is k-1 chained pairs)."""
    imgs, man = reference_images(width, height, stack)
    cores = os.cpu_count() or 1
    kind = "reference"
    try:
        sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
        import mtbalign as ref

        assert ref.kernels.engine_name() == "native"

        def run(workers):
            _, rec = ref.align_stack(imgs, levels=levels, tol=tol, workers=workers)
            return tuple(rec.cumulative[-1])
    except Exception:
        import mtb_oracle as orc

        kind, cores = "port", 1

        def run(workers):
            _, _, cum = orc.align_stack(imgs, levels, tol)
            return tuple(cum[-1])

    def best_of(workers):
        got = run(workers)  # warm-up
        times = []
        for _ in range(max(1, reps)):
            t0 = time.perf_counter()
            run(workers)
            times.append(time.perf_counter() - t0)
        return min(times), got, len(times)

    best, got, n = best_of(cores)
    best1, _, _ = best_of(1) if cores > 1 else (best, None, n)
    pairs = stack - 1
    what = "1 pair" if stack == 2 else f"1 {stack}-exposure stack ({pairs} chained pairs)"
    return {"value": pairs / best, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{what} {width}x{height} RGB8, {levels} levels, align_stack(workers={cores}), best of "
                      f"{n} after 1 warm-up; ms {best * 1e3:.1f}; last cumulative offset {got}",
            "workers_1": {"value": pairs / best1, "unit": UNIT, "ms": round(best1 * 1e3, 1)},
            "cpu_model": cpu_model()}


# ------------------------------------------------------------- our arm --
def make_inputs(torch, eng, units, stack, seed):
    """(units*stack, H, W, 3) device batch of synthetic exposure stacks (the
    SURVEY 8(d) recipe: synth.py generate_stack on a synthetic base; config 3
    uses the gains 2^((k-3)/3), gamma 1, max shift 20).  Returns the batch and
    each pair's ground-truth offset (target onto reference)."""
    from paper_2007_06483_b200.image import shift_rgb_device
    from paper_2007_06483_b200.synth import apply_lut_device, draw_manifest, synthetic_rgb_device, tone_lut

    h, w = eng.height, eng.width
    batch = torch.empty((stack * units, h, w, 3), dtype=torch.uint8, device="cuda")
    truth = []
    n_bases = min(units, 4)
    bases = [synthetic_rgb_device(seed + b, w, h) for b in range(n_bases)]
    for u in range(units):
        if stack == 2:
            pw, cum, gains, gammas = draw_manifest(2, seed=seed + u, max_shift=63)
        else:
            pw, cum, gains, gammas = draw_manifest(stack, seed=seed + u, max_shift=20,
                                                   gains=[2 ** ((k - 3) / 3) for k in range(stack)],
                                                   gammas=[1.0] * stack)
        base = bases[u % n_bases]
        for i in range(stack):
            moved = shift_rgb_device(base.unsqueeze(0), [(-cum[i].dx, -cum[i].dy)])[0]
            apply_lut_device(moved, tone_lut(gains[i], gammas[i]), out=batch[stack * u + i])
        mid = stack // 2 if stack > 2 else 0
        for i in range(stack):
            if i != mid:
                truth.append((cum[i].dx - cum[mid].dx, cum[i].dy - cum[mid].dy))
    torch.cuda.synchronize()
    return batch, truth


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2007_06483_b200 as mtb
    from paper_2007_06483_b200 import _lib

    dist = None
    if world > 1:
        import torch.distributed as dist

    eng = mtb.MtbEngine(args.width, args.height, args.levels, args.tol)
    n_img = args.pairs * args.stack
    pairs = unit_pairs(args.pairs, args.stack)
    P = len(pairs)
    batch, truth = make_inputs(torch, eng, args.pairs, args.stack, seed=1000 * rank + 1)
    pyr = eng.alloc(n_img)
    table = eng.maps_table(pyr, pairs)
    acc = torch.empty((P, eng.n, 2), dtype=torch.int32, device="cuda")
    errs = torch.empty((P, eng.n, 9), dtype=torch.int64, device="cuda")
    done = torch.empty((P, eng.n), dtype=torch.int32, device="cuda")
    chunk = args.chunk if args.chunk > 0 else n_img
    k1_images = chunk  # images per K1 launch: one persistent launch per preprocess chunk; each event pair brackets ONE launch
    stream = torch.cuda.current_stream()

    fused = args.mode == "fused"
    n_launch_fused = eng.fused_launches(n_img, pairs) if args.mode == "fused" else 0  # pipe.cu launches per step

    def step(ev=None):
        if fused:
            # ev: one (start, end) pair around the whole pipelined sequence
            if ev is not None:
                cs = torch.cuda.current_stream()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(cs)
            eng.align_fused(batch, pairs, pyr, acc, errs, done, count=False)
            if ev is not None:
                e.record(cs)
                ev.append((s, e, n_img))
            return
        # ev: optional list of (start, end) event pairs around each K1 (pyramid_hist) launch
        for c0 in range(0, n_img, chunk):
            c = min(chunk, n_img - c0)
            for i0 in range(c0, c0 + c, k1_images):
                k = min(k1_images, c0 + c - i0)
                if ev is not None:
                    cs = torch.cuda.current_stream()   # the capture stream inside torch.cuda.graph
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record(cs)
                    eng.pyramid_hist(batch, pyr, i0, k)
                    e.record(cs)
                    ev.append((s, e, k))
                else:
                    eng.pyramid_hist(batch, pyr, i0, k)
            eng.threshold_levels(pyr, c, c0, discard_gray=not args.keep_gray)
        eng.search_table(table, P, acc, errs, done, count=False)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    got = [tuple(a) for a in acc[:, 0].cpu().tolist()]
    correct = sum(int(g == t) for g, t in zip(got, truth))

    # One step = one CUDA graph replay (all launches of the step captured once,
    # K1 event pairs included, so the per-launch timing stays live).
    graph, graph_events = None, []
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        before = _lib.launch_count()
        with torch.cuda.graph(graph):
            step()
        launches_captured = _lib.launch_count() - before
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()

    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    k1_events = []
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        torch.cuda.nvtx.range_push("timed")
        start.record(stream)
        for _ in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                step(k1_events)
        end.record(stream)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
    if os.environ.get("MTB_PROFILE_RANGE") and graph is not None:
        # diagnostics: a profiler range of 4 whole steps (ncu --replay-mode
        # app-range --profile-from-start off) for the DRAM bytes of the real,
        # concurrent pipeline rather than of one serialised launch
        torch.cuda.profiler.start()
        for _ in range(4):
            graph.replay()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    if graph is not None:
        # Events cannot time kernels inside a graph replay: time each K1 launch
        # with events on an instrumented (python-launched) step right after the
        # timed region, same inputs and buffers.
        torch.cuda.synchronize()
        for _ in range(3):
            step(k1_events)
        torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    if graph is not None:
        # replays launch the captured kernels without passing through the
        # library's counter: count = launches captured per step x steps
        launches = (launches_captured) * args.steps
    elapsed = start.elapsed_time(end) / 1e3
    if dist is not None:
        from paper_2007_06483_b200.dist import max_over_ranks

        elapsed = max_over_ranks(elapsed, device="cuda")
        dist.barrier()
    k1_ms = [s.elapsed_time(e) for s, e, _ in k1_events]
    k1_imgs = [k for _, _, k in k1_events]

    total_pairs = P * args.steps * world
    value = total_pairs / elapsed
    img_bytes = 3 * args.width * args.height
    peak, peak_src = load_peak()
    k1_avg_s = statistics.fmean(k1_ms) / 1e3
    k1_bytes = statistics.fmean(k1_imgs) * img_bytes
    if fused:
        # the pipelined launches overlap (PDL): per-launch figures are the
        # sequence's time and RGB bytes divided by its launch count
        k1_avg_s /= n_launch_fused
        k1_bytes /= n_launch_fused
    achieved = k1_bytes / k1_avg_s / 1e9
    if fused:
        # pipe_kernel is 100 % of a fused step (ncu launch list, profiles/): its
        # achieved rate is the timed graph replays' algorithmic bytes / time
        achieved = n_img * img_bytes / (elapsed / args.steps) / 1e9
    traffic = (load_traffic("pipe_kernel", args.width, args.height,
                            _lib.load().mtb_align_fused_images_per_launch(args.width, args.height)) if fused else
               load_traffic("k1_rgb_pyramid_kernel", args.width, args.height, k1_images))
    step_gbs = value / world * (n_img * img_bytes / P) / 1e9   # algorithmic bytes per pair = the step's RGB / pairs

    # every benched pair re-checked on the CPU (reference engine when built)
    oracle = None if args.no_oracle_check else oracle_check(args, torch, batch, pairs, acc, errs)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, torch, eng, batch, pyr, table, acc, errs, done, pairs)
    with_out = None
    if fused and not args.no_e2e and args.stack == 2:
        with_out = run_with_output(args, torch, eng, batch, pyr, acc, errs, done, P)
    latency = single_pair_latency(torch, mtb, batch) if args.config == 2 and not args.no_e2e else None

    out = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": round(elapsed / args.steps * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": (f"{P} x {args.width * args.height / 1e6:.0f}MP ({args.width}x{args.height}) RGB8 exposure pairs per GPU per step, "
                                if args.stack == 2 else
                                f"{args.pairs} x {args.stack}-exposure {args.width * args.height / 1e6:.0f}MP ({args.width}x{args.height}) RGB8 stacks "
                                f"aligned to their middle exposure ({P} pairs) per GPU per step, ")
                               + f"{args.levels} levels, tol {args.tol} (BASELINE config {args.config}, batched)",
                   "baseline_config": args.config,
                   "width": args.width, "height": args.height, "levels": args.levels, "tol": args.tol,
                   "pairs_per_step_per_gpu": P, "preprocess_chunk_images": chunk, "k1_images_per_launch": k1_images,
                   "discard_gray": not args.keep_gray,
                   "l2": f"inputs {n_img * img_bytes / 1e9:.2f} GB per step per GPU > 126 MB L2; no flush needed",
                   "parallelism": f"batch-shard dp{world} (no collective)",
                   "launch": "cuda-graph replay per step" if graph is not None else "python launches",
                   "mode": args.mode,
                   "correct_offsets": f"{correct}/{P} match ground truth"},
        "oracle_match": oracle,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                     "kernel": (f"pipe_kernel (fused K1+K3+K4, {_lib.load().mtb_align_fused_images_per_launch(args.width, args.height)} image(s) per launch, "
                                f"{n_launch_fused} PDL launches per step = 100% of the step; achieved = step RGB bytes / timed step)") if fused else
                               f"k1_rgb_pyramid_kernel (K1: RGB->gray->pyramid->histograms, {k1_images} images/launch)",
                     "algorithmic_bytes_per_launch": k1_bytes, "avg_launch_ms": round(k1_avg_s * 1e3, 4),
                     "whole_step_gbs": round(step_gbs, 1), "whole_step_frac": round(step_gbs / peak, 4)},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if e2e is not None:
        out["e2e"] = e2e
    if with_out is not None:
        out["with_output"] = with_out
    if latency is not None:
        out["single_pair_latency"] = latency
    return out


def oracle_check(args, torch, batch, pairs, acc, errs):
    """Copy every benched pair back and run it through the reference's own
    engine (oracle/_ref, mtbalign 0.1.0 + its Cython kernels) on all host
    cores: offset and all 9 x n error counts must match.  Falls back to the
    numpy restatement (oracle/mtb_oracle.py) when the reference is not built.
    Exits non-zero on any mismatch."""
    import concurrent.futures as cf

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    t0 = time.perf_counter()
    try:
        sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
        import mtbalign as ref

        kind = "reference (oracle/_ref, native engine)"

        def pyr_of(img):
            return ref.build_mtb_pyramid(ref.build_pyramid(ref.to_grayscale(img), args.levels), args.tol)

        def search(a, b):
            r = ref.find_offset(a, b)
            return tuple(r.offset), {t.level: [e for _, e in t.candidates] for t in r.traces}
    except Exception:
        import mtb_oracle as orc

        kind = "port (oracle/mtb_oracle.py)"

        def pyr_of(img):
            return orc.preprocess(img, args.levels, args.tol)["mtb"]

        def search(a, b):
            r = orc.find_offset(a, b)
            return tuple(r["offset"]), {t["level"]: [e for _, e in t["candidates"]] for t in r["traces"]}

    acc_h, errs_h = acc.cpu().numpy(), errs.cpu().numpy()
    imgs_needed = sorted({i for p in pairs for i in p})
    # ranks of a multi-GPU run share the host's cores
    workers = max(1, (os.cpu_count() or 1) // int(os.environ.get("WORLD_SIZE", "1")))
    pyrs = {}
    with cf.ThreadPoolExecutor(max_workers=workers) as pool:
        futs = {}
        for i in imgs_needed:   # one image on the host at a time per worker slot
            futs[i] = pool.submit(pyr_of, batch[i].cpu().numpy())
            if len(futs) >= 2 * workers:
                for j, f in list(futs.items()):
                    pyrs[j] = f.result()
                futs = {}
        for j, f in futs.items():
            pyrs[j] = f.result()
        results = list(pool.map(lambda pq: search(pyrs[pq[0]], pyrs[pq[1]]), pairs))
    bad = []
    for q, (off, tr) in enumerate(results):
        ok = tuple(acc_h[q, 0].tolist()) == off and all(errs_h[q, k].tolist() == tr[k] for k in tr)
        if not ok:
            bad.append(q)
    line = {"matched": f"{len(pairs) - len(bad)}/{len(pairs)}", "checker": kind,
            "what": "offset + all 9 x levels candidate error counts of every benched pair",
            "seconds": round(time.perf_counter() - t0, 1)}
    if bad:
        print(json.dumps({"oracle_mismatch": bad[:16], **line}), file=sys.stderr, flush=True)
        raise SystemExit(f"oracle mismatch on pairs {bad[:16]}")
    return line


def single_pair_latency(torch, mtb, batch):
    """Paper-style one-pair alignment (config 2): get_exp_shift on one
    device-resident 24 MP pair, CUDA events, median of 10 after 3 warm-ups."""
    a, b = batch[0], batch[1]
    for _ in range(3):
        mtb.get_exp_shift(a, b)
    times = []
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        mtb.get_exp_shift(a, b)
        e.record()
        e.synchronize()
        times.append(s.elapsed_time(e))
    return {"ms_median": round(statistics.median(times), 4), "ms_best": round(min(times), 4),
            "api": "get_exp_shift (its own dispatch: staged kernels for one pair; device-resident pair, includes the offset readback)"}


def _world_max_time(dt):
    """(max over ranks of dt, world size): whole-job rates for multi-GPU runs."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        from paper_2007_06483_b200.dist import max_over_ranks

        dist.barrier()
        return max_over_ranks(dt, device="cuda"), dist.get_world_size()
    return dt, 1


def run_with_output(args, torch, eng, batch, pyr, acc, errs, done, P):
    """SURVEY 8(d) "with output": the step also writes every target aligned
    onto its reference (shift_rgb of image 2p+1 by pair p's offset, fill 0;
    image.py:82-93), read from and written to HBM: +6 W H bytes per pair."""
    from paper_2007_06483_b200 import _lib

    w, h = args.width, args.height
    out = torch.empty((P, h, w, 3), dtype=torch.uint8, device="cuda")
    pairs = [(2 * p, 2 * p + 1) for p in range(P)]
    stream = torch.cuda.current_stream()

    def step():
        eng.align_fused(batch, pairs, pyr, acc, errs, done, count=False)
        offs = acc[:, 0].contiguous()   # (P, 2) int32 on the device: no host round trip
        _lib.call("mtb_shift_rgb", batch[1].data_ptr(), 3 * w, 2 * 3 * w * h, w, h, P, offs.data_ptr(),
                  0, 0, 0, out.data_ptr(), 3 * w, 3 * w * h, stream.cuda_stream)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    steps = 20
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(steps):
        step()
    e.record(stream)
    torch.cuda.synchronize()
    dt = s.elapsed_time(e) / 1e3
    dt, nranks = _world_max_time(dt)
    return {"value": round(P * steps * nranks / dt, 2), "unit": UNIT,
            "bytes_per_pair": 12 * w * h, "note": "align_fused + shift_rgb of each target (device offsets), python launches"}


E2E_UNITS = 16   # e2e steps carry the first 16 units (pairs / stacks): PCIe-bound either way,
                 # and 8 ranks x a 64-pair pinned batch would pin 74 GB of host memory


def run_e2e(args, torch, eng, batch, pyr, table, acc, errs, done, pairs):
    """Same metric through the public engine API from pinned HOST buffers: every step
    copies the step's RGB pairs H2D and reads the offsets back D2H (timed)."""
    units = min(args.pairs, E2E_UNITS)
    pairs = unit_pairs(units, args.stack)
    batch = batch[:units * args.stack]
    P = len(pairs)
    host = torch.empty(batch.shape, dtype=torch.uint8, pin_memory=True)
    host.copy_(batch)
    out_host = torch.empty((P, 2), dtype=torch.int32, pin_memory=True)
    dev_in = torch.empty_like(batch)
    stream = torch.cuda.current_stream()

    fused = args.mode == "fused"

    def step():
        if fused:
            # H2D of image i overlaps the pipeline of the images before it
            eng.align_fused_host(host, pairs, pyr, acc, errs, done, dev=dev_in, count=False)
        else:
            dev_in.copy_(host, non_blocking=True)
            eng.preprocess(dev_in, pyr, count=False)
            eng.search_table(table_in, P, acc, errs, done, count=False)
        out_host.copy_(acc[:P, 0], non_blocking=True)

    table_in = eng.maps_table(pyr, pairs)
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(args.e2e_steps):
        step()
    e.record(stream)
    torch.cuda.synchronize()
    dt = s.elapsed_time(e) / 1e3
    dt, nranks = _world_max_time(dt)
    return {"value": round(P * args.e2e_steps * nranks / dt, 2), "unit": UNIT, "pairs_per_step": P,
            "h2d_bytes_per_step": int(host.numel()), "d2h_bytes_per_step": int(out_host.numel() * 4),
            "api": ("MtbEngine.align_fused_host (per-image H2D on a copy stream overlapped with the pipeline)"
                    if args.mode == "fused" else "MtbEngine.preprocess + search_table on an H2D-copied pinned batch")}


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch this command under
    torch.distributed.run with N ranks (one per GPU, 127.0.0.1 rendezvous);
    rank 0 prints the line."""
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        raise SystemExit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        cb = time_reference(args.width, args.height, args.levels, args.tol, args.cpu_reps, args.stack)
        line = {"metric": METRIC, "value": round(cb["value"], 4), "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.cpu_reps, "warmup": 1, "ms_per_step": round(1e3 / cb["value"], 2),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
                "data": "synthetic", "impl": "reference",
                "config": {"workload": (f"1 x {args.width * args.height / 1e6:.0f}MP ({args.width}x{args.height}) RGB8 pair per step, "
                                        if args.stack == 2 else
                                        f"1 x {args.stack}-exposure {args.width * args.height / 1e6:.0f}MP stack per step, ")
                                       + f"{args.levels} levels, tol {args.tol} (BASELINE config {args.config})"},
                "cpu_baseline": cb,
                "e2e": {"value": round(cb["value"], 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    if world > 1:
        import torch.distributed as dist

        if torch.cuda.device_count() < world:
            raise SystemExit(f"--gpus {world} needs {world} visible GPUs; {torch.cuda.device_count()} present")
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        torch.cuda.set_device(0)
    out = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = time_reference(args.width, args.height, args.levels, args.tol, args.cpu_reps,
                                                 args.stack)
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
