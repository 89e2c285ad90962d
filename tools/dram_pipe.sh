B="python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --no-e2e --pairs 8 --mode fused"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:pipe -s 30 -c 8 --csv --log-file gpurun_out/dram_pipe.csv $B > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/dram_pipe.csv")) if len(r)>10]
h=rows[0]; data={}
for r in rows[1:]:
    d=dict(zip(h,r)); data.setdefault(d["ID"],{})[d["Metric Name"]]=d["Metric Value"]
for i,m in data.items(): print(i, {k: round(float(v)/1e6,1) for k,v in m.items()})
PY
grep -i "pass" gpurun_out/dram_pipe.csv | head -3
