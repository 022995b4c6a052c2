# ncu --set full of one select_kernel launch at c3 (after warm-up)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"select_kernel" -s 4 -c 1 -o gpurun_out/prof_select_c3 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_select_c3.log 2>&1
tail -3 gpurun_out/ncu_select_c3.log
