"""Workload for compute-sanitizer (tools/sanitize.sh): a fused batch of 8
images (4 K1 launches of 2 images + trailing search launches), chain pairs
plus a cross-launch pair, then the streamed-input variant (per-image H2D
flags), then a staged preprocess + search of the same batch (64 pairs too:
the per-pair coarse-level search), then the on-chip cluster preprocess
(csrc/cluster.cu) at its natural cluster size and forced to 8 CTAs."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06483_b200 as mtb  # noqa: E402
from paper_2007_06483_b200.synth import generate_stack, synthetic_rgb_device  # noqa: E402

w, h = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (512, 384)
imgs, _ = generate_stack(synthetic_rgb_device(1, w, h), 8, seed=1, max_shift=12)
batch = torch.stack(imgs).contiguous()
pairs = [(i, i + 1) for i in range(7)] + [(0, 7)]
eng = mtb.MtbEngine(w, h, 6, 4)
print("launches", eng.fused_launches(8, pairs))
_, acc, _ = eng.align_fused(batch, pairs)
host = batch.cpu().pin_memory()
_, _, acc2, _ = eng.align_fused_host(host, pairs)
pyr = eng.preprocess(batch)
acc3, _ = eng.search(pyr, pairs)
acc64, _ = eng.search(pyr, pairs * 8)
outs = []
for forced in (None, "8"):
    if forced:
        os.environ["MTB_CM_CLUSTER"] = forced
    if eng.maps_cluster() or forced:
        p2 = eng.alloc(8, gray=False)
        eng.preprocess_maps(batch, p2)
        outs.append(eng.search(p2, pairs)[0])
    os.environ.pop("MTB_CM_CLUSTER", None)
torch.cuda.synchronize()
assert torch.equal(acc, acc2) and torch.equal(acc, acc3) and torch.equal(acc64[:8], acc)
assert all(torch.equal(o, acc) for o in outs), len(outs)
print("ok", acc[:, 0].tolist(), "on-chip runs", len(outs))
