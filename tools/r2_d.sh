#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -u -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider --timeout 60 > gpurun_out/r2d_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2d_tests.txt
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 200 $B > gpurun_out/r2d_bench_res.log 2>&1
MTB_LIB_PATH=$PWD/paper_2007_06483_b200/_lib/exp/nosearch.so timeout 200 $B > gpurun_out/r2d_bench_ns.log 2>&1
MTB_LIB_PATH=$PWD/paper_2007_06483_b200/_lib/exp/nosearch.so timeout 300 ncu --set full --clock-control none --import-source on -k regex:res_kernel -s 2 -c 1 -o gpurun_out/r2d_nosearch python bench.py --steps 1 --warmup 1 --no-graph --no-e2e --no-cpu-baseline --pairs 8 > gpurun_out/r2d_ncu_ns.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:res_kernel -s 2 -c 1 -o gpurun_out/r2d_res python bench.py --steps 1 --warmup 1 --no-graph --no-e2e --no-cpu-baseline --pairs 8 > gpurun_out/r2d_ncu.log 2>&1
tail -2 gpurun_out/r2d_tests.txt; for f in res ns; do grep -o '"ms_per_step": [0-9.]*\|correct_offsets": "[^"]*' gpurun_out/r2d_bench_$f.log; done
