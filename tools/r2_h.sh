#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=$PWD/paper_2007_06483_b200/_lib/exp
for n in base l1na ld128 loadsonly nohist; do
MTB_RES_TRACE=gpurun_out/r2h_$n.bin MTB_LIB_PATH=$L/tr_$n.so timeout 120 python bench.py --steps 1 --warmup 1 --no-graph --no-e2e --no-cpu-baseline --pairs 8 > gpurun_out/r2h_$n.log 2>&1
done
