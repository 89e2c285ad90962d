for P in 16 32 64; do
echo "pairs=$P $(timeout 200 python bench.py --mode fused --pairs $P --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["config"]["correct_offsets"])')"
done
