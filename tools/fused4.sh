timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | grep -E "passed|failed|Error|assert" | head -8
python tools/pipe_trace.py 2>&1 | tail -12
B="python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --no-e2e --pairs 8 --mode fused"
ncu --set full --import-source on --clock-control none -k regex:pipe -s 30 -c 1 -o gpurun_out/pipe4 -f $B > gpurun_out/ncu_pipe4.log 2>&1
tail -1 gpurun_out/ncu_pipe4.log
