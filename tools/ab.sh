# A/B: current build vs exp/$1.so, alternating
for i in 1 2; do
for lib in paper_2007_06483_b200/_lib/libmtbalign_b200.so paper_2007_06483_b200/_lib/exp/$1.so; do
 echo "$(basename $lib): $(MTB_LIB_PATH=$PWD/$lib timeout 120 python bench.py --mode fused --steps 40 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])')"
done; done
