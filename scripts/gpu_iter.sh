# one optimisation iteration: parity suite, smoke, select breakdown, benches (c2, c3)
set -x
timeout 700 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 240 -rf -x > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -2 gpurun_out/smoke.log
CSATTN_PHASE_PROF=1 timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/phase_c3.json 2> gpurun_out/phase_c3.err
CSATTN_PHASE_PROF=1 timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/phase_c2.json 2> gpurun_out/phase_c2.err
grep csattn gpurun_out/phase_c3.err gpurun_out/phase_c2.err
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
tail -n 2 gpurun_out/bench_c2.err gpurun_out/bench_c3.err
python scripts/summ.py gpurun_out/bench_c2.json gpurun_out/bench_c3.json
