#!/bin/bash
# select change: GPU suites (default, forced retry, no split) + c3/c2 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x > gpurun_out/sel_tests.log 2>&1
tail -2 gpurun_out/sel_tests.log
CSATTN_SPEC_KEEP=1.6 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_sharding.py -m gpu -q -p no:cacheprovider --timeout 600 -x > gpurun_out/sel_tests_retry.log 2>&1
tail -1 gpurun_out/sel_tests_retry.log
CSATTN_NO_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -p no:cacheprovider --timeout 600 -x > gpurun_out/sel_tests_nosplit.log 2>&1
tail -1 gpurun_out/sel_tests_nosplit.log
for cfg in c3 c2; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/sel_$cfg.json 2> gpurun_out/sel_$cfg.err
done
python scripts/summ.py gpurun_out/sel_c3.json gpurun_out/sel_c2.json
