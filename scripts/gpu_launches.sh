# per-kernel launch list (ncu gpu__time_duration, cold/serialised) for a config: $1 tag $2 config
T=${1:-l}; CFG=${2:-c2}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 40 --csv \
  --log-file gpurun_out/${T}_launches_${CFG}.csv python bench.py --config ${CFG} --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_launches_${CFG}.log 2>&1
echo "ncu rc=$?"
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/${T}_launches_${CFG}.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
for r in rows[1:]:
    print(r[ki][:60], r[vi])
PY
