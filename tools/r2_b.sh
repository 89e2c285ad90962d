#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for t in $(python -m pytest tests/test_gpu_fused.py --collect-only -q 2>/dev/null | grep "::"); do
  timeout 60 python -u -m pytest "$t" -x -q -p no:cacheprovider > /tmp/t.log 2>&1; rc=$?
  echo "$rc $t $(tail -1 /tmp/t.log)" >> gpurun_out/r2b_tests.txt
  if [ $rc -ne 0 ]; then tail -30 /tmp/t.log >> gpurun_out/r2b_tests.txt; fi
done
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 200 $B > gpurun_out/r2b_bench_res.log 2>&1
MTB_LIB_PATH=$PWD/paper_2007_06483_b200/_lib/exp/nosearch.so timeout 200 $B > gpurun_out/r2b_bench_nosearch.log 2>&1
MTB_LIB_PATH=$PWD/paper_2007_06483_b200/_lib/exp/sw4.so timeout 200 $B > gpurun_out/r2b_bench_sw4.log 2>&1
cat gpurun_out/r2b_tests.txt
for f in res nosearch sw4; do echo $f; grep -o '"ms_per_step": [0-9.]*\|correct_offsets": "[^"]*' gpurun_out/r2b_bench_$f.log; done
