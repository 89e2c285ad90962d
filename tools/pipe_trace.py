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
J = 2 * P + 1 + eng.n
G = torch.cuda.get_device_properties(0).multi_processor_count
tr = torch.zeros(J * G * 16, dtype=torch.int64, device="cuda")
for it in range(4):
    if it == 3:
        os.environ["MTB_PIPE_TRACE"] = str(tr.data_ptr())
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    eng.align_fused(batch, pairs, pyr, count=False)
    e.record()
    torch.cuda.synchronize()
    print("step ms", s.elapsed_time(e))
t = tr.view(J, G, 16).cpu().numpy().astype(np.int64)
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

# stragglers: per CTA aux durations in K1 launches 10..30
aux = (t[10:31, :, 5] - t[10:31, :, 4]) / 1e3
k1a = (t[10:31, :, 3] - t[10:31, :, 1]) / 1e3
sm = t[10:31, :, 6]
print("aux per CTA: median over launches, top 12 slow CTAs (cta, smid, aux_med, k1aux_med)")
rot = int(os.environ.get("MTB_PIPE_ROT", "0"))
if rot:
    slice_of = np.array([[(c + rot * j) % G for c in range(G)] for j in range(10, 31)])
    aux_s = np.zeros(G)
    for jj in range(aux.shape[0]):
        aux_s[slice_of[jj]] = aux[jj]
    print("by slice (last launch): slowest slices", np.argsort(-aux_s)[:5], "by SM:", [int(sm[-1, c]) for c in np.argsort(-aux[-1])[:5]])
    print("per launch slowest (cta, slice, smid):", [(int(np.argmax(aux[jj])), int(slice_of[jj][np.argmax(aux[jj])]), int(sm[jj, np.argmax(aux[jj])]), round(float(aux[jj].max()),1)) for jj in range(0, 21, 3)])
med = np.median(aux, axis=0)
order = np.argsort(-med)
for c in order[:12]:
    print(c, int(sm[0, c]), round(float(med[c]), 1), round(float(np.median(k1a[:, c])), 1))
print("fast CTAs", [(int(c), int(sm[0, c]), round(float(med[c]), 1)) for c in order[-6:]])
print("corr of aux time between consecutive launches", np.corrcoef(aux[:-1].ravel(), aux[1:].ravel())[0, 1])

print("phase start offsets (us after aux start) for CTA 147 vs CTA 5, launches 20..23; phases 0..6, then aux end")
for j in range(20, 24):
    for c in (147, 5):
        r = t[j, c]
        ph = [round((r[8 + p] - r[4]) / 1e3, 1) if r[8 + p] else None for p in range(7)]
        print(j, c, ph, round((r[5] - r[4]) / 1e3, 1))
