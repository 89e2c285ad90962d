"""Timeline of the fused pipeline from per-CTA %globaltimer stamps (MTB_PIPE_TRACE)."""
import os, sys
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_06483_b200 as mtb
from bench import make_inputs

P = int(os.environ.get("PAIRS", "16"))
eng = mtb.MtbEngine(6000, 4000, 6, 4)
batch, truth = make_inputs(torch, eng, P, seed=1)
pairs = [(2 * p, 2 * p + 1) for p in range(P)]
pyr = eng.alloc(2 * P)
J = eng.fused_launches(2 * P, pairs)
G = torch.cuda.get_device_properties(0).multi_processor_count
tr = torch.zeros(J * G * 80, dtype=torch.int64, device="cuda")
for it in range(4):
    if it == 3:
        os.environ["MTB_PIPE_TRACE"] = str(tr.data_ptr())
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    eng.align_fused(batch, pairs, pyr, count=False)
    e.record()
    torch.cuda.synchronize()
    print("step ms", s.elapsed_time(e))
t = tr.view(J, G, 80).cpu().numpy().astype(np.int64)
t0 = t[0, :, 0].min()
print("launch  k1_start(min,max) k1_tiles flush k1_aux k1_end_max | aux_start(min,max) aux  aux_end_max   (us; medians over CTAs)")
for j in range(J):
    r = t[j]
    has_k1 = (r[:, 1] > 0).all()
    def us(x):
        return (x - t0) / 1e3
    line = f"{j:4d} "
    if has_k1:
        line += (f"{us(r[:, 0]).min():8.1f} {us(r[:, 0]).max():8.1f} {np.median((r[:, 1] - r[:, 0]) / 1e3):6.1f} "
                 f"{np.median((r[:, 2] - r[:, 1]) / 1e3):5.1f} {np.median((r[:, 3] - r[:, 2]) / 1e3):5.1f} "
                 f"{us(r[:, 3]).max():8.1f} | ")
    else:
        line += " " * 49 + "| "
    line += (f"{us(r[:, 4]).min():8.1f} {us(r[:, 4]).max():8.1f} {np.median((r[:, 5] - r[:, 4]) / 1e3):6.1f} "
             f"{us(r[:, 5]).max():8.1f}  aux max {((r[:, 5] - r[:, 4]) / 1e3).max():5.1f}")
    print(line)

# phase starts (first task of each aux phase in the CTA) relative to the CTA's K1 start, launches 20..23
names = {6: "search", 0: "K3 L0", 1: "K3 L1", 2: "K3 L2", 3: "K3 L3", 4: "L4-5", 5: "pad"}
for j in range(20, 24):
    r = t[j]
    row = []
    for p in (6, 0, 1, 2, 3, 4):
        v = r[:, 8 + p]
        ok = v > 0
        row.append(f"{names[p]} {np.median((v[ok] - r[ok, 0]) / 1e3):6.1f}" if ok.any() else f"{names[p]}   -  ")
    end = np.median((np.maximum(r[:, 3], r[:, 5]) - r[:, 0]) / 1e3)
    print(j, " | ".join(row), f"| end {end:6.1f} | k1 tiles end {np.median((r[:, 1] - r[:, 0]) / 1e3):6.1f}")
    pro = [np.median((r[:, i] - r[:, 0]) / 1e3) for i in (4, 5, 6, 7)]
    print("   aux prologue: start %.1f  med_ready %.1f  consts %.1f  done %.1f" % tuple(pro))
