# mixed-mode select: tests + c3 bench
T=${1:-tail}
timeout 900 python -m pytest tests/test_gpu_select_tail.py tests/test_gpu_scale.py tests/test_gpu_parity.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/${T}_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err; echo "bench rc=$?"
python scripts/summ.py gpurun_out/${T}_bench_c3.json
CSATTN_TAIL_SPLIT=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_c3_notail.json 2>/dev/null; echo "bench notail rc=$?"
python scripts/summ.py gpurun_out/${T}_bench_c3_notail.json
