# full GPU check: suites (default, forced speculation misses, no split), facade,
# benches c2/c3 (+ c4, c5 when FULL=1)
set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x > gpurun_out/gpu_tests.log 2>&1
tail -2 gpurun_out/gpu_tests.log
CSATTN_SPEC_KEEP=1.6 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_sharding.py -m gpu -q -p no:cacheprovider --timeout 600 -x > gpurun_out/gpu_tests_forced_retry.log 2>&1
tail -2 gpurun_out/gpu_tests_forced_retry.log
CSATTN_NO_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -p no:cacheprovider --timeout 600 -x > gpurun_out/gpu_tests_nosplit.log 2>&1
tail -2 gpurun_out/gpu_tests_nosplit.log
timeout 600 tests/cpp/test_facade > gpurun_out/facade.log 2>&1; tail -1 gpurun_out/facade.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python scripts/summ.py gpurun_out/bench_c2.json gpurun_out/bench_c3.json
if [ "$FULL" = "1" ]; then
  timeout 1200 python bench.py --config c4 --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
  timeout 1500 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
  for f in gpurun_out/bench_c4.json gpurun_out/bench_c5.json; do python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['value'], d['e2e']['value'], d['setup_s'])" $f; done
fi
