# ncu --set full of select_kernel and attend128 at c3 (one launch each) + launch list: $1 = tag
T=${1:-n3}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'select_kernel|attend128' -s 8 -c 2 \
  -o gpurun_out/${T}_c3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
