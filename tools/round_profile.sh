# full default bench + launch list + full ncu capture of the fused pipe kernel (round evidence)
# pipe launches per step at the default 64 pairs: J = 71 (2 images per launch); --warmup 3 -> step 3 starts at launch 213
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpuinfo.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
B="python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-e2e --no-oracle-check"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pipe -s 213 -c 71 --csv --log-file gpurun_out/launches.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --cache-control none -k regex:pipe -s 245 -c 2 -o gpurun_out/pipe_full -f $B > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
