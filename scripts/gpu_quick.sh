# quick GPU check: $1 = tag; parity-critical GPU tests, c3 bench, phase profile
T=${1:-q}
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hardening.py tests/test_gpu_sharding.py -x -q > gpurun_out/${T}_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${T}_gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err; echo "bench c3 rc=$?"
CSATTN_PHASE_PROF=1 timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/${T}_phase_c3.json 2> gpurun_out/${T}_phase_c3.err; echo "phase rc=$?"
grep csattn gpurun_out/${T}_phase_c3.err
python scripts/summ.py gpurun_out/${T}_bench_c3.json
