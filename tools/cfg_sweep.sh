for lib in paper_2007_06483_b200/_lib/libmtbalign_b200.so paper_2007_06483_b200/_lib/exp/g4s2.so; do
 echo "$lib: $(MTB_LIB_PATH=$PWD/$lib timeout 120 python bench.py --mode fused --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["config"]["correct_offsets"])')"
done
MTB_LIB_PATH=$PWD/paper_2007_06483_b200/_lib/exp/g4s2.so timeout 150 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -1
