"""Config 3: a 7 x 24 MP exposure stack aligned to its middle
exposure (pivot 3, 6 pairs), device-resident batch, fused engine vs staged
engine; CUDA-event timing over repeated calls (stack-level throughput)."""
import os, sys
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_06483_b200 as mtb
from paper_2007_06483_b200.synth import synthetic_rgb_device

W, H, N, P = 6000, 4000, 7, 3
eng = mtb.MtbEngine(W, H, 6, 4)
base = synthetic_rgb_device(2, W, H)
batch = torch.stack([base] * N).contiguous()
pairs = [(P, i) for i in range(N) if i != P]
pyr = eng.alloc(N)


def run(fn, reps=30):
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


fused_ms = run(lambda: eng.align_fused(batch, pairs, pyr, count=False))
table = eng.maps_table(pyr, pairs)
staged_ms = run(lambda: (eng.preprocess(batch, pyr, count=False), eng.search_table(table, len(pairs), count=False)))
print(f"config 3 (7 x 24 MP, pivot, 6 pairs): fused {fused_ms:.3f} ms/stack = {6 / fused_ms * 1e3:.0f} pairs/s; "
      f"staged {staged_ms:.3f} ms/stack = {6 / staged_ms * 1e3:.0f} pairs/s; "
      f"algorithmic 84 MB/pair -> fused {6 * 84e6 / (fused_ms / 1e3) / 1e9:.0f} GB/s")
