# K1 probe: full / stream-only / compute-only launch times (bench's live K1 events)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for pr in 0 1 2; do
  echo "probe=$pr $(MTB_K1_PROBE=$pr timeout 300 python bench.py --steps 50 --no-cpu-baseline --no-e2e $BENCH_ARGS 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["value"], d["ms_per_step"], r["avg_launch_ms"], r["achieved"], r["frac"])')"
done
