for m in staged fused staged fused; do
echo "$m $(timeout 120 python bench.py --mode $m --steps 100 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["config"]["correct_offsets"], d["roofline"]["frac"])')"
done
