T=${1:-c2}
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q > gpurun_out/${T}_fused.log 2>&1; echo "fused tests rc=$?"; tail -2 gpurun_out/${T}_fused.log
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err; echo "bench c2 rc=$?"
python scripts/summ.py gpurun_out/${T}_bench_c2.json
