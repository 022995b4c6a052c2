set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_info2.txt
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_kernel|insert_kernel" --csv --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c2_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 4 -c 1 -o gpurun_out/prof_decode_c2 python bench.py --config c2 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_c2.log 2>&1
tail -3 gpurun_out/bench_c2.err gpurun_out/bench_c3.err
