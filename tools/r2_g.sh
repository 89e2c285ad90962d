#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=$PWD/paper_2007_06483_b200/_lib/exp
MTB_RES_TRACE=gpurun_out/r2g_trace_ns.bin MTB_LIB_PATH=$L/trace_ns.so timeout 200 python bench.py --steps 1 --warmup 1 --no-graph --no-e2e --no-cpu-baseline --pairs 8 > gpurun_out/r2g_trace_ns.log 2>&1
MTB_LIB_PATH=$L/nosearch.so timeout 300 ncu --set full --clock-control none --import-source on -k regex:res_kernel -s 2 -c 1 -o gpurun_out/r2g_nosearch python bench.py --steps 1 --warmup 1 --no-graph --no-e2e --no-cpu-baseline --pairs 8 > gpurun_out/r2g_ncu_ns.log 2>&1
