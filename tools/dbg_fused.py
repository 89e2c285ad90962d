import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import mtb_oracle as orc
import paper_2007_06483_b200 as mtb
imgs = [np.full((96, 128, 3), v, np.uint8) for v in (0, 0, 255, 255, 77, 77)]
eng = mtb.MtbEngine(128, 96, 6, 4)
rgb = torch.from_numpy(np.stack(imgs)).cuda()
for trial in range(2):
    pyr = eng.alloc(6)
    pyr.mtb.fill_(7); pyr.excl.fill_(7)
    pyr, acc, errs = eng.align_fused(rgb, [(0, 1), (2, 3), (4, 5)], pyr=pyr)
    torch.cuda.synchronize()
    print("medians", pyr.medians.cpu().numpy().tolist())
    for i in range(6):
        for k in range(eng.n):
            m = eng.bitmap_words(pyr.mtb, i, k).cpu().numpy().view(np.uint64)
            e = eng.bitmap_words(pyr.excl, i, k).cpu().numpy().view(np.uint64)
            pre = orc.preprocess(imgs[i], 6, 4)
            em = orc.pack(pre["mtb"][k]["mtb"]); ee = orc.pack(pre["mtb"][k]["excl"])
            if not (np.array_equal(m, em) and np.array_equal(e, ee)):
                print("img", i, "level", k, "mtb bad rows", np.nonzero((m != em).any(1))[0][:10], "excl bad rows", np.nonzero((e != ee).any(1))[0][:10])
                print(" got", [hex(x) for x in e[:4, 0]], "want", [hex(x) for x in ee[:4, 0]])
