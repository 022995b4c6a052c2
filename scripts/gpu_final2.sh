# round-end evidence, part 2: gpu_final.sh + the reference arm + ncu captures
# (c3 select/attend, c2 fused step) + c2 launch list: $1 = tag
T=${1:-fin2}
bash scripts/gpu_final.sh $T
timeout 1200 python bench.py --impl reference > gpurun_out/${T}_bench_ref_c3.json 2> /dev/null; echo "ref rc=$?"; tail -c 300 gpurun_out/${T}_bench_ref_c3.json
bash scripts/gpu_ncu_c3.sh ${T}n
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'fused_step' -s 8 -c 1 \
  -o gpurun_out/${T}_c2 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c2.csv \
  python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches c2 rc=$?"
