# union attend at c3: launch durations of one step's kernels + one full capture of attend_range_kernel
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:"union|range|tail|attend|select|route|insert" -s 40 -c 40 --log-file gpurun_out/launches_union_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_union.log 2>&1
tail -2 gpurun_out/ncu_launches_union.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attend_tc_kernel" -s 2 -c 1 -o gpurun_out/prof_tc_c3 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_range.log 2>&1
tail -2 gpurun_out/ncu_range.log
