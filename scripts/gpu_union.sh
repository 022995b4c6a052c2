# union attend check: fork-batch parity, full parity suite, c3 with/without union
set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 240 -rf -x -k union > gpurun_out/union_test.log 2>&1
tail -3 gpurun_out/union_test.log
CSATTN_UNION=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3_nounion.json 2> gpurun_out/bench_c3_nounion.err
tail -n 3 gpurun_out/bench_c3.err
python scripts/summ.py gpurun_out/bench_c3.json gpurun_out/bench_c3_nounion.json
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x > gpurun_out/gpu_tests.log 2>&1
tail -2 gpurun_out/gpu_tests.log
