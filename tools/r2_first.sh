#!/usr/bin/env bash
# Round-2 first look at the resident kernel: smoke, fused parity tests, A/B bench vs pipe.cu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2a_smoke.log
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q > gpurun_out/r2a_fused.log 2>&1; echo "fused rc=$?" >> gpurun_out/r2a_fused.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2a_bench_res.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_bench_res.log
MTB_FUSED_IMPL=pipe timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2a_bench_pipe.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_bench_pipe.log
tail -5 gpurun_out/r2a_smoke.log gpurun_out/r2a_fused.log; tail -c 1500 gpurun_out/r2a_bench_res.log; tail -c 600 gpurun_out/r2a_bench_pipe.log
