#!/usr/bin/env python3
"""Executed warp instructions and stall samples per CUDA source line of one
kernel: joins an ncu capture's per-SASS-address counts (--page source
--print-source sass) with the line table nvdisasm prints for the same build
(-lineinfo).  With --smem: shared-memory wavefronts and excessive (bank
conflict) wavefronts per line instead, sorted by excess.  Usage:
    python tools/ncu_lines.py REPORT.ncu-rep LIB.so MANGLED_KERNEL [top] [--smem]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

smem = "--smem" in sys.argv
argv = [x for x in sys.argv if x != "--smem"]
rep, lib, kern = argv[1], os.path.abspath(argv[2]), argv[3]
top = int(argv[4]) if len(argv) > 4 else 40

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    data.append(dict(zip(hdr, r)))
base = int(data[0]["Address"], 16)

with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=d, capture_output=True)
    cubins = [f for f in os.listdir(d) if f.endswith(".cubin")]
    sass = ""
    for f in cubins:
        t = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, f)], capture_output=True, text=True).stdout
        if f".text.{kern}:" in t:
            sass = t
            break
start = sass.index(f".text.{kern}:")
line_of = {}
cur = None
for ln in sass[start:].splitlines()[1:]:
    if ln.startswith(".text.") or ln.startswith("\t.section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur

cnt, smp = collections.Counter(), collections.Counter()
wf, wfx = collections.Counter(), collections.Counter()
for d in data:
    off = int(d["Address"], 16) - base
    key = line_of.get(off, ("?", 0))
    cnt[key] += int(d["Instructions Executed"] or 0)
    smp[key] += int(d["Warp Stall Sampling (All Samples)"] or 0)
    wf[key] += int(d.get("L1 Wavefronts Shared") or 0)
    wfx[key] += int(d.get("L1 Wavefronts Shared Excessive") or 0)
if smem:
    tw, tx = sum(wf.values()), sum(wfx.values())
    print(f"{tw:,} shared wavefronts, {tx:,} excessive ({100 * tx / max(tw, 1):.1f} %)")
    for key, n in wfx.most_common(top):
        print(f"{n:>12,} excess {wf[key]:>12,} total  {key[0]}:{key[1]}")
    sys.exit(0)
tot, tots = sum(cnt.values()), sum(smp.values())
print(f"{tot:,} warp instructions, {tots:,} samples")
for key, n in cnt.most_common(top):
    print(f"{100 * n / tot:5.1f}% inst {100 * smp[key] / max(tots, 1):5.1f}% samples  {key[0]}:{key[1]}")
