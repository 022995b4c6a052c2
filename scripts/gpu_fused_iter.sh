T=${1:-fz}
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q > gpurun_out/${T}_fused.log 2>&1; echo "fused tests rc=$?"; tail -2 gpurun_out/${T}_fused.log
for c in c2 c4; do
CSATTN_FZ_DEBUG=1 timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err; echo "bench $c rc=$?"
grep "\[fz\]" gpurun_out/${T}_bench_$c.err | tail -2
done
python scripts/summ.py gpurun_out/${T}_bench_c2.json gpurun_out/${T}_bench_c4.json
