"""A/B of the small-image preprocess paths on one GPU: staged (K1 +
hist_median + threshold through a gray arena) vs on-chip (csrc/cluster.cu),
N images of W x H, CUDA-event timing; prints one JSON line.
Usage: python tools/cluster_ab.py [W H N]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_06483_b200 as mtb  # noqa: E402
from paper_2007_06483_b200.synth import synthetic_rgb_device  # noqa: E402

W, H, N = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (1024, 768, 1024)
eng = mtb.MtbEngine(W, H, 6, 4)
base = torch.stack([synthetic_rgb_device(i, W, H) for i in range(8)])
batch = base.repeat((N + 7) // 8, 1, 1, 1)[:N].contiguous()
staged = eng.alloc(N)
onchip = eng.alloc(N, gray=False)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


t_st = timed(lambda: eng.preprocess(batch, staged, count=False))
t_oc = timed(lambda: eng.preprocess_maps(batch, onchip))
same = bool(torch.equal(staged.medians, onchip.medians))
for k in range(eng.n):
    nw64, off = int(eng.geom[k, 4]), int(eng.geom[k, 5])
    sl = slice(off, off + nw64 * int(eng.geom[k, 1]))
    same &= bool(torch.equal(staged.mtb[:, sl], onchip.mtb[:, sl]) and torch.equal(staged.excl[:, sl], onchip.excl[:, sl]))
rgb = 3 * W * H * N
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
print(json.dumps({"w": W, "h": H, "n_img": N, "cluster": eng.maps_cluster(),
                  "staged_ms": round(t_st, 4), "onchip_ms": round(t_oc, 4), "speedup": round(t_st / t_oc, 3),
                  "onchip_rgb_gbs": round(rgb / t_oc / 1e6, 1), "onchip_frac": round(rgb / t_oc / 1e6 / peak, 4),
                  "identical": same}))
