for lib in paper_2007_06483_b200/_lib/libmtbalign_b200.so paper_2007_06483_b200/_lib/exp/evlast.so; do
 echo "$(basename $lib): $(MTB_LIB_PATH=$PWD/$lib timeout 120 python bench.py --mode fused --steps 40 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["config"]["correct_offsets"])')"
done
B="python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --no-e2e --pairs 8 --mode fused"
MTB_LIB_PATH=$PWD/paper_2007_06483_b200/_lib/exp/evlast.so ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:pipe -s 30 -c 4 --csv --log-file gpurun_out/dram_ev.csv $B > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/dram_ev.csv")) if len(r)>10]
h=rows[0]; data={}
for r in rows[1:]:
    d=dict(zip(h,r)); data.setdefault(d["ID"],{})[d["Metric Name"]]=d["Metric Value"]
for i,m in data.items(): print("evlast", i, {k: round(float(v)/1e6,1) for k,v in m.items()})
PY
