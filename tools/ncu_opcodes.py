#!/usr/bin/env python3
"""Executed-SASS opcode histogram of the FIRST kernel in an ncu capture
(--page source --print-source sass) -> markdown.
    python tools/ncu_opcodes.py REPORT.ncu-rep "title" > profiles/<tag>_sass_histogram.md"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    data.append(dict(zip(hdr, r)))
dyn, stat, special = collections.Counter(), collections.Counter(), collections.Counter()
for d in data:
    src = d["Source"].strip()
    if not src:
        continue
    toks = src.split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    n = int(d["Instructions Executed"] or 0)
    dyn[op.split(".")[0]] += n
    stat[op.split(".")[0]] += 1
    if re.match(r"(UTMALDG|UBLKCP|SYNCS|ATOMS|CCTL|MEMBAR|RED|ATOMG|LDGSTS|IDP|VABSDIFF4|POPC|FENCE)", op):
        special[op] += n
tot = sum(dyn.values())
print(f"# SASS opcode histogram — {title}\n")
print("Dynamic: warp-level instructions executed in ONE mid-step pipe_kernel launch (K1 of 2 images of 24 MP")
print("plus that launch's K3 and search tasks), from the ncu `--set full` capture; static: instructions in the")
print("kernel's SASS.  Blackwell-native evidence: UTMALDG (TMA tensor loads), UBLKCP (bulk copies), SYNCS")
print("(mbarriers), ATOMS.POPC.INC (aggregated shared-memory histogram increments).\n")
print(f"Total executed: {tot:,} warp instructions ({tot / 2 / 1e6:.1f} M per image).\n")
print("| opcode | executed | % | static |\n|---|---:|---:|---:|")
for op, n in dyn.most_common(40):
    print(f"| {op} | {n:,} | {100 * n / tot:.1f} | {stat[op]} |")
print("\nSelected opcodes with modifiers:\n\n| opcode | executed |\n|---|---:|")
for op, n in sorted(special.items(), key=lambda kv: -kv[1]):
    print(f"| {op} | {n:,} |")
