# K1 variant matrix: library x probe -> K1 avg launch ms (32 images)
run() { MTB_LIB_PATH=$1 MTB_K1_PROBE=$2 timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e $BENCH_ARGS 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["value"], r["avg_launch_ms"], r["frac"])'; }
for lib in paper_2007_06483_b200/_lib/libmtbalign_b200.so ${EXP_LIBS:-paper_2007_06483_b200/_lib/exp/*.so}; do
  for pr in 0 2; do echo "$(basename $lib) probe=$pr $(run $PWD/$lib $pr)"; done
done
