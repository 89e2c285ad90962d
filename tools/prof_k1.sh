B="python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --no-e2e --pairs 4"
ncu --set full --import-source on --clock-control none -k regex:k1_rgb -s 4 -c 1 -o gpurun_out/k1b -f $B > gpurun_out/ncu_k1b.log 2>&1
tail -3 gpurun_out/ncu_k1b.log
