# union attend: parity test, profiled timeline, c3 bench
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 240 -rf -x -k union > gpurun_out/union_test.log 2>&1
tail -1 gpurun_out/union_test.log
bash scripts/gpu_union_prof.sh
CSATTN_UNION=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python scripts/summ.py gpurun_out/bench_c3.json
