set -x
timeout 700 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 240 -x > gpurun_out/gpu_tests.log 2>&1
CSATTN_SPEC_KEEP=1.6 timeout 700 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -p no:cacheprovider --timeout 240 -x > gpurun_out/gpu_tests_forced_retry.log 2>&1
tail -2 gpurun_out/gpu_tests_forced_retry.log
tail -2 gpurun_out/gpu_tests.log
CSATTN_NO_SPLIT=1 timeout 700 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -p no:cacheprovider --timeout 240 -x > gpurun_out/gpu_tests_nosplit.log 2>&1
tail -2 gpurun_out/gpu_tests_nosplit.log
timeout 600 tests/cpp/test_facade > gpurun_out/facade.log 2>&1; tail -1 gpurun_out/facade.log
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
tail -n 2 gpurun_out/bench_c2.err gpurun_out/bench_c3.err
python scripts/summ.py gpurun_out/bench_c2.json gpurun_out/bench_c3.json
