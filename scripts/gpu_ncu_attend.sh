# ncu --set full of one attend_kernel launch and one insert/route launch at c3
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"attend_kernel|route_kernel|insert_kernel" -s 12 -c 3 -o gpurun_out/prof_attend_c3 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_attend_c3.log 2>&1
tail -3 gpurun_out/ncu_attend_c3.log
# launch list of a whole bench command (per-kernel durations, cold/serialised)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_c3.log 2>&1
tail -2 gpurun_out/ncu_launches_c3.log
