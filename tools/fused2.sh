timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 50 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("value", d["value"], "ms", d["ms_per_step"], d["config"]["correct_offsets"])'
B="python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --no-e2e --pairs 8"
ncu --set full --import-source on --clock-control none -k regex:pipe -s 30 -c 1 -o gpurun_out/pipe3 -f $B > gpurun_out/ncu_pipe3.log 2>&1
tail -1 gpurun_out/ncu_pipe3.log
