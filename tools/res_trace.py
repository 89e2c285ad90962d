"""Summarise a resident-kernel trace (experiment build -DRES_EXP_TRACE, MTB_RES_TRACE=path):
per image the spread of CTA arrive times, the barrier-to-medians latency and the step period."""
import sys
import numpy as np
d = open(sys.argv[1], "rb").read()
n_img, G = np.frombuffer(d[:8], dtype=np.int32)
t = np.frombuffer(d[8:], dtype=np.uint64).reshape(n_img, G, 8).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1e3, np.nan)   # us
for s in range(n_img):
    st, ar, md, k3, l4, l5, c6, c7 = (t[s, :, i] for i in range(8))
    print(f"   flushed-flag seen {np.nanmin(c6):8.1f}..{np.nanmax(c6):8.1f}  arrive2 {np.nanmin(l4):8.1f}..{np.nanmax(l4):8.1f}  medians broadcast {np.nanmax(l5):8.1f}")
    print(f"img {s:3d} start {np.nanmin(st):8.1f}..{np.nanmax(st):8.1f}  arrive {np.nanmin(ar):8.1f}..{np.nanmax(ar):8.1f} "
          f"(med {np.nanmedian(ar):8.1f})  medians {np.nanmin(md):8.1f}..{np.nanmax(md):8.1f}  k3done {np.nanmin(k3):8.1f}..{np.nanmax(k3):8.1f}")
ar = np.nanmax(t[:, :, 1], axis=1)
print("step period (last arrive to last arrive) us:", np.round(np.diff(ar), 1))
