# DRAM bytes of 4 whole bench steps as they really run (concurrent PDL launches, graph replay)
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum
MTB_PROFILE_RANGE=1 timeout 600 ncu --replay-mode app-range --clock-control none --cache-control none --metrics $M --csv --log-file gpurun_out/range_dram.csv python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-oracle-check "$@" > gpurun_out/range_bench.log 2>&1
cat gpurun_out/range_dram.csv | tail -8
