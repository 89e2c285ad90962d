B="python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --no-e2e --pairs 8 --mode fused"
ncu --set full --import-source on --clock-control none --cache-control none -k regex:pipe -s 30 -c 1 -o gpurun_out/pipe6 -f $B > gpurun_out/ncu_pipe6.log 2>&1
tail -1 gpurun_out/ncu_pipe6.log
