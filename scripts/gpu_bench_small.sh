# c2 / c4 benches (fused cluster step by default) + the c3 default: $1 tag
T=${1:-s}
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${T}_gpu_tests.log
for c in c2 c4; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err; echo "bench $c rc=$?"
done
CSATTN_FUSED=0 timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/${T}_bench_c2_nofused.json 2> gpurun_out/${T}_bench_c2_nofused.err; echo "c2 nofused rc=$?"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err; echo "bench c3 rc=$?"
python scripts/summ.py gpurun_out/${T}_bench_c2.json gpurun_out/${T}_bench_c2_nofused.json gpurun_out/${T}_bench_c4.json gpurun_out/${T}_bench_c3.json
