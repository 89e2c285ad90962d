B="python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --no-e2e --pairs 8 --mode fused"
ncu --set full --import-source on --clock-control none --cache-control none -k regex:pipe -s 30 -c 2 -o gpurun_out/pnow -f $B > /dev/null 2>&1
ls gpurun_out/pnow*
