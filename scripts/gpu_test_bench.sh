# GPU round: parity suite, smoke, benches (c2, c3). Outputs under gpurun_out/.
set -x
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 240 -rf -x > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
tail -n 3 gpurun_out/bench_c2.err gpurun_out/bench_c3.err
