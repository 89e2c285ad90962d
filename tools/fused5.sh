timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | grep -E "passed|failed|Error|assert" | head -8
B="python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --no-e2e --pairs 8 --mode fused"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --cache-control none --clock-control none -k regex:pipe -s 25 -c 6 --csv --log-file gpurun_out/pipe_nf.csv $B > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/pipe_nf.csv")) if len(r)>10]
h=rows[0]; data={}
for r in rows[1:]:
    d=dict(zip(h,r)); data.setdefault(d["ID"],{})[d["Metric Name"]]=d["Metric Value"]
for i,m in data.items(): print(i, m)
PY
