# quick throughput sweep of bench knobs (no cpu baseline / e2e)
for c in 0 2 4 8; do
  echo "chunk=$c $(timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-e2e --chunk $c 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"])')"
done
echo "keep-gray chunk=2 $(timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-e2e --chunk 2 --keep-gray 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])')"
