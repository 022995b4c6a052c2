# speculative-cut checks: parity suite with forced retries, then benches
set -x
CSATTN_SPEC_KEEP=1.6 timeout 700 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 240 -x > gpurun_out/gpu_tests_forced_retry.log 2>&1
tail -2 gpurun_out/gpu_tests_forced_retry.log
CSATTN_SPEC_KEEP=0 timeout 700 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 240 -x > gpurun_out/gpu_tests_nospec.log 2>&1
tail -2 gpurun_out/gpu_tests_nospec.log
bash scripts/gpu_iter.sh
timeout 600 tests/cpp/test_facade > gpurun_out/facade.log 2>&1; tail -2 gpurun_out/facade.log
