# GPU iteration: $1 = tag. Full GPU test suite, c3 + c2 bench (no CPU legs),
# ncu launch list + a full capture of select at c3.
T=${1:-iter}
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${T}_gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err; echo "bench c3 rc=$?"
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err; echo "bench c2 rc=$?"
python - <<PY
import json
for c in ("c3","c2"):
    try:
        d=json.loads(open("gpurun_out/${T}_bench_%s.json"%c).read().strip().splitlines()[-1])
        k=d["roofline"]["kernels"]
        print(c, "step", round(d["value"],1), "e2e", round(d["e2e"]["value"],1), "select", round(k["select"]["ms"]*1e3,1), "attend", round(k["attend"]["ms"]*1e3,1), "insert", round(k["insert"]["ms"]*1e3,1), "frac", round(d["roofline"]["frac"],3))
    except Exception as e: print(c, "ERR", e)
PY
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'select_kernel' -s 4 -c 1 \
  -o gpurun_out/${T}_sel python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
fi
