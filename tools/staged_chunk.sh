for c in 1 2 0; do
echo "chunk=$c $(timeout 300 python bench.py --mode staged --steps 50 --no-cpu-baseline --no-e2e --chunk $c 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])')"
done
B="python bench.py --mode staged --steps 1 --warmup 3 --no-graph --no-cpu-baseline --no-e2e --pairs 4 --chunk 1"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/staged_c1.csv $B > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/staged_c1.csv")) if len(r)>10]
h=rows[0]; data={}
for r in rows[1:]:
    d=dict(zip(h,r)); data.setdefault(d["ID"],{"name":d["Kernel Name"][:30]})[d["Metric Name"]]=d["Metric Value"]
ids=sorted(data, key=int)
for i in ids[-16:]:
    m=data[i]; print(i, m["name"], m["gpu__time_duration.sum"], int(float(m["dram__bytes_read.sum"]))//1000000, int(float(m["dram__bytes_write.sum"]))//1000000)
PY
