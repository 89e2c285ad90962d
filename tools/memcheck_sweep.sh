#!/usr/bin/env bash
# compute-sanitizer memcheck with torch caching disabled (exact allocation bounds) over the fused, staged
# and on-chip paths at several geometries; prints each run's errors and summary.
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
CS="/usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 5"
run() { echo "== $*"; timeout 900 $CS "$@" 2>&1 | grep -E "Invalid|ERROR SUMMARY|at .*\.cu:" | head -8; }
run python tools/sanitize.py
run python tools/sanitize.py 1000 700
run python bench.py --pairs 2 --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline --no-oracle-check
run python bench.py --config 4 --pairs 2 --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline --no-oracle-check
run python bench.py --config 1 --pairs 16 --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline --no-oracle-check
run python bench.py --config 3 --pairs 1 --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline --no-oracle-check
