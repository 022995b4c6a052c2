CSATTN_UNION=1 CSATTN_UNION_PROF=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_uprof.json 2> gpurun_out/bench_c3_uprof.err
grep "union kernel\|tile " gpurun_out/bench_c3_uprof.err
