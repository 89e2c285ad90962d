"""Phase timeline of the on-chip preprocess (csrc/cluster.cu) from an
experiment build with -DCM_TRACE (tools/build_exp.sh cmtrace -DCM_TRACE;
run with MTB_LIB_PATH=paper_2007_06483_b200/_lib/exp/cmtrace.so).
Prints the launch shape and mean per-image phase durations (us) over the
first 8 images of the first 256 CTAs.  Usage: python tools/cluster_trace.py [W H N]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_06483_b200 as mtb  # noqa: E402
from paper_2007_06483_b200 import _lib  # noqa: E402
from paper_2007_06483_b200.synth import synthetic_rgb_device  # noqa: E402

W, H, N = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (1024, 768, 1024)
lib = _lib.load()
shape = (ctypes.c_int * 4)()
lib.mtb_preprocess_maps_shape(W, H, 6, shape)
eng = mtb.MtbEngine(W, H, 6, 4)
batch = torch.stack([synthetic_rgb_device(i, W, H) for i in range(8)]).repeat((N + 7) // 8, 1, 1, 1)[:N].contiguous()
pyr = eng.alloc(N, gray=False)
for _ in range(3):
    eng.preprocess_maps(batch, pyr)
torch.cuda.synchronize()
tr = np.zeros((256, 8, 6), dtype=np.uint64)
fn = lib.mtb_cm_trace
fn.argtypes = [ctypes.c_void_p]
fn(tr.ctypes.data)
C, G, tpc, nq = list(shape)
ctas = min(256, nq * C)
t = tr[:ctas].astype(np.int64)
t0 = t[:, 0, 0].min()
names = ["A (tiles)", "A' (L4/5)", "B push+barrier", "B gather+median", "C threshold", "next image gap"]
print(f"shape C={C} G={G} tpc={tpc} clusters={nq} ctas={ctas}")
d = np.diff(t, axis=2) / 1e3                     # [cta, img, 5]
gap = (t[:, 1:, 0] - t[:, :-1, 5]) / 1e3          # end of image j -> start of j+1
for i, n in enumerate(names[:5]):
    print(f"{n:18s} mean {d[:, 1:, i].mean():6.2f} us   p90 {np.percentile(d[:, 1:, i], 90):6.2f}")
print(f"{names[5]:18s} mean {gap.mean():6.2f} us")
per = (t[:, 7, 5] - t[:, 1, 0]) / 6e3
print(f"per image (images 1..6) {per.mean():6.2f} us; first image start spread {(t[:, 0, 0] - t0).max() / 1e3:.2f} us")
