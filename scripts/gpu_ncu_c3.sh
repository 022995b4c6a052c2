# ncu --set full of one select, attend, route and insert launch at c3 + the launch list
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"select_kernel|attend128|route_kernel|insert_kernel" -s 20 -c 5 -o gpurun_out/prof_c3 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1
tail -2 gpurun_out/ncu_c3.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_c3.log 2>&1
tail -1 gpurun_out/ncu_launches_c3.log
