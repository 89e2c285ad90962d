# A/B at another geometry: tools/ab_cfg.sh EXP W H PAIRS
for i in 1 2; do
for lib in paper_2007_06483_b200/_lib/libmtbalign_b200.so paper_2007_06483_b200/_lib/exp/$1.so; do
 echo "$(basename $lib) $2x$3: $(MTB_LIB_PATH=$PWD/$lib timeout 120 python bench.py --mode fused --width $2 --height $3 --pairs $4 --steps 40 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])')"
done; done
