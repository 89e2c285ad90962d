# ncu captures for K1/K3/K4 hotspots (source-level) and cross-kernel L2 behaviour
set -x
B="python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --no-e2e --pairs 4"
ncu --set full --import-source on --clock-control none -k regex:k1_rgb -s 4 -c 1 -o gpurun_out/k1 -f $B > gpurun_out/ncu_k1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:threshold_levels -s 2 -c 1 -o gpurun_out/k3 -f $B > gpurun_out/ncu_k3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:level_search -s 17 -c 1 -o gpurun_out/k4 -f $B > gpurun_out/ncu_k4.log 2>&1
for c in 0 2; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --cache-control none --clock-control none --csv --log-file gpurun_out/chunk$c.csv python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --no-e2e --pairs 8 --chunk $c > /dev/null 2>&1
done
ls -la gpurun_out
