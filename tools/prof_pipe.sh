B="python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --no-e2e --pairs 8"
ncu --set full --import-source on --clock-control none -k regex:pipe -s 30 -c 1 -o gpurun_out/pipe2 -f $B > gpurun_out/ncu_pipe2.log 2>&1
tail -1 gpurun_out/ncu_pipe2.log
