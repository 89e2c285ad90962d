# other BASELINE configs (not the headline): config 1 (1024x768 pairs) and config 4 (4000x3000 pairs)
for m in fused staged; do
  echo "cfg1 $m: $(timeout 300 python bench.py --width 1024 --height 768 --pairs 512 --steps 20 --mode $m --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])')"
  echo "cfg4 $m: $(timeout 300 python bench.py --width 4000 --height 3000 --pairs 32 --steps 50 --mode $m --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])')"
done
