"""Per-SM occupancy of the fused pipeline: CTA entry/exit stamps (%globaltimer, %smid)
from MTB_PIPE_TRACE; gaps between consecutive CTAs on one SM = launch turnover cost."""
import os, sys
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_06483_b200 as mtb
from bench import make_inputs

P = int(os.environ.get("PAIRS", "32"))
W, H = int(os.environ.get("W", "6000")), int(os.environ.get("H", "4000"))
eng = mtb.MtbEngine(W, H, 6, 4)
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
sm, t_in, t_out = t[:, :, 16], t[:, :, 17], t[:, :, 18]
t0 = t_in.min()
span = (t_out.max() - t0) / 1e3
dur = (t_out - t_in) / 1e3
print(f"span {span:.1f} us, launches {J}, {span / J:.2f} us/launch")
print(f"CTA duration us: median {np.median(dur):.1f}  p10 {np.percentile(dur, 10):.1f}  p90 {np.percentile(dur, 90):.1f}")
gaps, busy = [], []
for s_ in range(G):
    m = sm == s_
    ins, outs = np.sort(t_in[m]), np.sort(t_out[m])
    busy.append((outs - ins).sum() / 1e3)
    gaps.extend(((ins[1:] - outs[:-1]) / 1e3).tolist())
gaps = np.array(gaps)
print(f"per-SM busy fraction: mean {np.mean(busy) / span:.3f}  min {np.min(busy) / span:.3f}")
print(f"CTA turnover gap us: median {np.median(gaps):.2f}  p90 {np.percentile(gaps, 90):.2f}  max {gaps.max():.2f}")
# per launch: first entry, last entry, first exit, last exit (relative)
for j in range(J // 2 - 2, J // 2 + 3):
    print(j, "entry %.1f..%.1f  exit %.1f..%.1f  dur med %.1f" % ((t_in[j].min() - t0) / 1e3, (t_in[j].max() - t0) / 1e3,
          (t_out[j].min() - t0) / 1e3, (t_out[j].max() - t0) / 1e3, np.median(dur[j])))

# inside a CTA (launches 10..J-10, medians over CTAs), us from entry
mid = slice(10, J - 10)
rel = lambda x: np.median((x[mid] - t_in[mid]) / 1e3)
print("first K1 tile ready %.2f | K1 loop end (warp 0) %.2f | exit %.2f" % (rel(t[:, :, 21]), rel(t[:, :, 1]), rel(t_out)))
we = t[:, :, 24:40]
print("warp drain end (median over CTAs) :", " ".join("%.1f" % np.median((we[mid, :, w] - t_in[mid]) / 1e3) for w in range(16)))
idle = ((t_out[mid, :, None] - we[mid]) / 1e3)
print("warp idle at CTA end us: mean per warp %.2f (K1 warps %.2f, aux warps %.2f)" % (idle.mean(), idle[..., :12].mean(), idle[..., 12:].mean()))
print("spin ns per CTA: search deps %.0f  thresholds %.0f  gray slot %.0f" % tuple(np.median(t[mid, :, i]) for i in (19, 20, 22)))
wmax = we.max(axis=2)
print("exit - last warp end us: median %.2f p90 %.2f" % (np.median((t_out[mid] - wmax[mid]) / 1e3), np.percentile((t_out[mid] - wmax[mid]) / 1e3, 90)))
print("last warp end - first warp end us: median %.2f" % np.median((wmax[mid] - we.min(axis=2)[mid]) / 1e3))
# the slowest warp of each CTA: its last task's phase and duration
ls, lp = t[:, :, 40:56], t[:, :, 56:72]
arg = we.argmax(axis=2)
import collections
ph = collections.Counter()
durs = collections.defaultdict(list)
for j in range(10, J - 10):
    for c in range(G):
        w = arg[j, c]
        ph[int(lp[j, c, w])] += 1
        durs[int(lp[j, c, w])].append((we[j, c, w] - ls[j, c, w]) / 1e3)
names = {6: "search", 0: "K3 L0", 1: "K3 L1", 2: "K3 L2", 3: "K3 L3", 4: "L4-5", 5: "pad"}
print("slowest warp's last task:", ", ".join(f"{names.get(k, k)} {v} (med {np.median(durs[k]):.2f} us)" for k, v in ph.most_common()))
# all warps: last task phase distribution and duration
allp = collections.Counter(lp[10:J - 10].ravel().tolist())
print("all warps' last task:", ", ".join(f"{names.get(k, k)} {v}" for k, v in allp.most_common()))
