"""Summarise an ncu report: headline metrics + SASS instruction/stall buckets by execution count."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
for x in r[1:]:
    d = dict(zip(h, x))
    n = d["Metric Name"]
    if any(k in n for k in ["Duration", "DRAM Throughput", "Issue Slots", "L2 Hit", "Executed Instructions", "No Eligible"]):
        print(d["Section Name"][:25], "|", n, "|", d["Metric Value"], d["Metric Unit"])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:]]
tot = sum(int(d["Instructions Executed"]) for d in data)
stall = sum(int(d["Warp Stall Sampling (All Samples)"]) for d in data)
print("total", tot, "samples", stall, "n", len(data))
b, bs, bn = collections.Counter(), collections.Counter(), collections.Counter()
for d in data:
    c = int(d["Instructions Executed"])
    b[c] += c
    bs[c] += int(d["Warp Stall Sampling (All Samples)"])
    bn[c] += 1
print("count  n_instr  warp_instr  stall_samples")
for c, v in sorted(b.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(c, bn[c], v, bs[c])
print("top stalls")
for i, d in sorted(enumerate(data), key=lambda x: -int(x[1]["Warp Stall Sampling (All Samples)"]))[:12]:
    print(i, d["Warp Stall Sampling (All Samples)"].rjust(5), d["Instructions Executed"].rjust(8), d["Source"][:80])
