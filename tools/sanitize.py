"""Workload for compute-sanitizer (tools/sanitize.sh): a fused batch of 8
images (4 K1 launches of 2 images + trailing search launches), chain pairs
plus a cross-launch pair, then the streamed-input variant (per-image H2D
flags), then a staged preprocess + search of the same batch."""
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
torch.cuda.synchronize()
assert torch.equal(acc, acc2) and torch.equal(acc, acc3)
print("ok", acc[:, 0].tolist())
