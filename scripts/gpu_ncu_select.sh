# ncu --set full of select_kernel and insert_kernel at c3 (one launch each, after warm-up)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"select_kernel|insert_kernel" -s 6 -c 2 -o gpurun_out/prof_select_c3 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_select_c3.log 2>&1
tail -3 gpurun_out/ncu_select_c3.log
