# attend variants at c3: $1 = tag, $2.. = CSATTN_ATT_GR values
T=$1; shift
CSATTN_ATT_GR=44 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -k "lockstep or attend or c3 or c2" > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${T}_tests.log
for g in "$@"; do
  CSATTN_ATT_GR=$g timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/${T}_bench_$g.json 2>/dev/null; echo "gr=$g rc=$?"
  python scripts/summ.py gpurun_out/${T}_bench_$g.json
done
