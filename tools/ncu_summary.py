#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (run in the build container).

    python tools/ncu_summary.py --full gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
        --tag r1 --out profiles

Writes profiles/ncu_summary.json (per-kernel DRAM bytes per launch from the
--set full capture; bench.py reads it for roofline.traffic) and a readable
profiles/<tag>_ncu.md with the launch list shares and the full-set metrics.
"""

import argparse
import io
import collections
import csv
import json
import os
import subprocess

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("mtb::", "")}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    v = float(v) * SCALE.get(units[i], 1)
                except ValueError:
                    pass
                d[m] = v
        res.append(d)
    return res


def launch_list(path):
    rows = [r for r in csv.DictReader(l for l in open(path) if not l.startswith("=="))]
    agg = collections.OrderedDict()
    for r in rows:
        k = r["Kernel Name"].split("(")[0].replace("void ", "").replace("mtb::", "")
        t = float(r["Metric Value"].replace(",", "")) / 1e3  # ns -> us
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
    return agg, len(rows)


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return {}
    d = dict(zip(r[0], r[2]))
    pre = "smsp__pcsamp_warps_issue_stalled_"
    res = {}
    for k, v in d.items():
        if k.startswith(pre) and not k.endswith("not_issued"):
            try:
                res[k[len(pre):]] = float(v.replace(",", ""))
            except ValueError:
                pass
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--out", default="profiles")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    fm = full_metrics(a.full)
    per_kernel = collections.OrderedDict()
    for d in fm:
        per_kernel.setdefault(d["kernel"], []).append(d)
    # merge with an existing summary: kernels captured earlier keep their entries
    path = os.path.join(a.out, "ncu_summary.json")
    summary = {"source": os.path.basename(a.full), "tag": a.tag, "kernels": {}, "detail": {}}
    if os.path.exists(path):
        with open(path) as f:
            old = json.load(f)
        summary["kernels"].update(old.get("kernels", {}))
        summary["detail"].update(old.get("detail", {}))
        for key in ("by_workload", "by_workload_note"):   # bench.py's roofline.traffic lookup
            if key in old:
                summary[key] = old[key]
    for k, ds in per_kernel.items():
        traffic = [d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in ds]
        summary["kernels"][k] = round(sum(traffic) / len(traffic))
        summary["detail"][k] = ds
    with open(os.path.join(a.out, "ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    lines = [f"# ncu summary {a.tag}", "", a.note, "", "## --set full (per launch; cold caches, clocks not locked)", "",
             "| kernel | grid | time us | DRAM read MB | DRAM write MB | DRAM % | SM % | warps act % | issue % | inst |",
             "|---|---|---:|---:|---:|---:|---:|---:|---:|---:|"]
    for d in fm:
        lines.append("| {kernel} | {g} | {t:.1f} | {r:.1f} | {w:.1f} | {dp:.1f} | {sp:.1f} | {wa:.1f} | {ia:.1f} | {ins:.0f} |".format(
            kernel=d["kernel"], g=d.get("launch__grid_size", ""), t=d["gpu__time_duration.sum"],
            r=d["dram__bytes_read.sum"] / 1e6, w=d["dram__bytes_write.sum"] / 1e6,
            dp=d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"],
            sp=d["sm__throughput.avg.pct_of_peak_sustained_elapsed"],
            wa=d["sm__warps_active.avg.pct_of_peak_sustained_active"],
            ia=d["smsp__issue_active.avg.pct_of_peak_sustained_active"], ins=d["smsp__inst_executed.sum"]))
    st = stalls(a.full)
    if st:
        lines += ["", "## warp-state samples (first captured launch; % of samples)", "",
                  "| reason | % |", "|---|---:|"]
        tot = sum(st.values())
        for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:10]:
            lines.append(f"| {k} | {100 * v / tot:.1f} |")
    if a.launches:
        agg, n = launch_list(a.launches)
        tot = sum(v[1] for v in agg.values())
        lines += ["", f"## launch list ({n} launches, gpu__time_duration.sum, serialised, cold)", "",
                  "| kernel | launches | total us | share |", "|---|---:|---:|---:|"]
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| {k} | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
    with open(os.path.join(a.out, f"{a.tag}_ncu.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
