# staged path: chunk sweep at config 2 and config 4
for c in 0 2 4 8 16; do
  echo "cfg2 staged chunk $c: $(timeout 300 python bench.py --mode staged --chunk $c --steps 30 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])')"
done
for c in 0 4 8; do
  echo "cfg4 staged chunk $c: $(timeout 300 python bench.py --width 4000 --height 3000 --mode staged --chunk $c --steps 30 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])')"
done
