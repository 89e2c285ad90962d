#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -u -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider --timeout 60 > gpurun_out/r2k_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2k_tests.txt
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 200 $B > gpurun_out/r2k_bench_res.log 2>&1
L=$PWD/paper_2007_06483_b200/_lib/exp
MTB_RES_TRACE=gpurun_out/r2k_trace_ns.bin MTB_LIB_PATH=$L/trace_ns.so timeout 200 python bench.py --steps 1 --warmup 1 --no-graph --no-e2e --no-cpu-baseline --pairs 8 > gpurun_out/r2k_trace_ns.log 2>&1
MTB_RES_TRACE=gpurun_out/r2k_trace.bin MTB_LIB_PATH=$L/trace.so timeout 200 python bench.py --steps 1 --warmup 1 --no-graph --no-e2e --no-cpu-baseline --pairs 8 > gpurun_out/r2k_trace.log 2>&1
tail -3 gpurun_out/r2k_tests.txt; grep -o '"ms_per_step": [0-9.]*\|correct_offsets": "[^"]*' gpurun_out/r2k_bench_res.log
