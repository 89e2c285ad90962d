"""Config 5 (BASELINE.json): one 1-gigapixel (40000 x 25000) RGB8 pair, 10
levels.  On ONE GPU: the staged engine (one K1 launch over the 6 GB pair,
thresholds, 10-level device search) with CUDA-event timing, and the
row-sharded phases driven as W virtual shards (loopback; serial on one GPU,
so this times the per-shard work, not a multi-GPU run).  Prints one JSON
line.  The 8-GPU row-sharded run uses sharded.align_pair_distributed under
torchrun (tests/test_gpu_sharded.py::test_nccl_row_sharded_when_two_gpus)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_06483_b200 as mtb  # noqa: E402
from paper_2007_06483_b200.image import shift_rgb_device  # noqa: E402
from paper_2007_06483_b200.sharded import align_pair_loopback  # noqa: E402
from paper_2007_06483_b200.synth import synthetic_rgb_device  # noqa: E402

W, H, L = 40000, 25000, 10
batch = torch.empty((2, H, W, 3), dtype=torch.uint8, device="cuda")
batch[0].copy_(synthetic_rgb_device(5, W, H))
shift_rgb_device(batch[0].unsqueeze(0), [(-301, 177)], out=batch[1].unsqueeze(0))
eng = mtb.MtbEngine(W, H, L, 4)
pyr = eng.alloc(2)
table = eng.maps_table(pyr, [(0, 1)])


def staged():
    eng.preprocess(batch, pyr, count=False)
    return eng.search_table(table, 1, count=False)


def timed(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        out = fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps, out


ms, (acc, _) = timed(staged, 10)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
byts = 2 * 3 * W * H
del pyr
torch.cuda.empty_cache()
lb_ms, res = timed(lambda: align_pair_loopback(batch[0], batch[1], 8, levels=L), 3)
print(json.dumps({
    "config": "BASELINE config 5: one 40000x25000 RGB8 pair, 10 levels, 1 B200",
    "staged_ms_per_pair": round(ms, 3), "staged_pairs_per_s": round(1e3 / ms, 1),
    "algorithmic_bytes_per_pair": byts, "staged_gbs": round(byts / ms / 1e6, 1),
    "staged_frac_of_hbm_peak": round(byts / ms / 1e6 / peak, 4),
    "offset": acc[0, 0].tolist(),
    "loopback_8_shards_ms_per_pair": round(lb_ms, 3),
    "loopback_offset": list(res.offset),
    "note": "loopback runs the 8 shards' phases serially on one GPU (host-driven, no overlap); "
            "per-shard work of the 8-GPU run is ~1/8 of the staged pair",
}))
